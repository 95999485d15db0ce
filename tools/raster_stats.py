"""Tuning diagnostic (not product code): one C2 (or C3) training step with the
raster kernels built with -DBS_RASTER_STATS; prints how the backward's kept
(warp, splat) iterations split by contributing lanes.  Run after
`BS_NVCC_EXTRA=-DBS_RASTER_STATS python -m paper_2512_20017_b200.build -f`."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2512_20017_b200 import _native, scenes
from paper_2512_20017_b200.culling import zorder_group
from paper_2512_20017_b200.trainer import SplatTrainer

model = sys.argv[1] if len(sys.argv) > 1 else "3dgs"
seed, n = (1, 1_000_000) if model == "3dgs" else (2, 2_000_000)
ds = scenes.generate_aerial_scene(seed, n, (1, 1), 8, 50.0, (1920, 1080))
g = zorder_group(ds.cloud, G=2048)
params = scenes.init_gaussians(g.sorted_cloud, seed, scenes.mean_spacing(50.0, (1, 1), n))
gt = scenes.synthetic_gt(seed, 8, 1920, 1080)
tr = SplatTrainer(params, g.group_begin(), g.aabbs.reshape(-1, 6), ds.views, gt=gt, model=model)
lib = C.CDLL(_native.lib_path())
out = (C.c_ulonglong * 64)()
tr.step([0, 3, 4, 7])
torch.cuda.synchronize()
lib.bs_debug_raster_stats(out, 1)
tr.step([0, 3, 4, 7])
torch.cuda.synchronize()
lib.bs_debug_raster_stats(out, 1)
s = np.array(out[:], dtype=np.float64)
print("instances", tr.last["n_inst"])
print(f"bwd warp-chunks {s[0]:.0f} kept iterations {s[1]:.0f} (per chunk {s[1]/max(s[0],1):.2f})")
print(f"  zero {s[2]/s[1]:.3f} sparse {s[3]/s[1]:.3f} dense {s[4]/s[1]:.3f} mean contributing lanes {s[5]/s[1]:.2f} mean live lanes {s[6]/s[1]:.2f}")
h = s[8:41]
print("  hist contributing lanes:", " ".join(f"{i}:{h[i]/s[1]:.3f}" for i in range(33)))
print(f"fwd warp-chunks {s[48]:.0f} kept iterations {s[49]:.0f}, lanes in support per kept iteration {s[50]/max(s[49],1):.2f}")
print(f"fused: warps {s[57]:.0f}, kept per warp {s[58]/max(s[57],1):.1f}, lists wrapped (> 128) {s[56]/max(s[57],1):.4f}, "
      f"> 192 {s[59]/max(s[57],1):.4f}, > 256 {s[60]/max(s[57],1):.4f}")
