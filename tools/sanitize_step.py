"""One small run of every kernel family of the step, for compute-sanitizer
(racecheck / memcheck / synccheck): 3DGS and 2DGS training
steps with multi-chunk groups (cp.async SH staging, G_SP clearing in the
projection), the radix binning pipeline, the tile-bucket sorts of every size
class, the standalone projection backward and Adam, selective Adam, the
fused raster kernel (kept lists in shared memory and their wrap-around
fallback) beside the separate forward / backward kernels, densification."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np
import torch

from paper_2512_20017_b200 import _native as nat
from paper_2512_20017_b200 import scenes
from paper_2512_20017_b200.trainer import AdamConfig, SplatTrainer

from _scene import c1_setup

torch.cuda.set_device(0)
ds, params, gb, aabb, gt = c1_setup(G=1000, n_points=4000, image_size=(96, 64))
lr = scenes.lr_table(50.0)
for model in ("3dgs", "2dgs"):
    for selective in (False, True):
        tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, model=model, adam=AdamConfig(lr, selective=selective))
        for b in ([0, 3, 5], [1, 2, 6]):
            tr.step(b)
        torch.cuda.synchronize()
        print(model, "selective" if selective else "dense", "ok", tr.last["n_rows"], tr.last["n_inst"], flush=True)
# separate raster kernels (the default 3DGS step runs the fused one), and the
# fused kernel's wrap-around fallback (large splats: > 128 kept per warp)
tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, adam=AdamConfig(lr))
tr.raster_fused = False
tr.step([0, 3, 5])
big = params.copy()
big[1, :, :3] += np.float32(1.5)
tr = SplatTrainer(big, gb, aabb, ds.views, gt=gt, adam=AdamConfig(lr), bg=(0.1, 0.2, 0.3))
tr.step([2, 6])
# densification (statistic in the fused backward, mark / apply / AABBs)
tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, adam=AdamConfig(lr))
tr.track_densify_stats(True)
tr.step([0, 3, 5])
from paper_2512_20017_b200.trainer import DensifyConfig
st = tr.densify_stats.cpu().numpy()
rep = tr.densify(DensifyConfig(grad_threshold=float(np.median(st[:, 0] / np.maximum(st[:, 1], 1))), split_scale=1.0,
                               min_opacity=0.05))
tr.step([1, 4])
torch.cuda.synchronize()
print("separate raster, fused fallback, densify ok", rep["n_before"], rep["n_after"], flush=True)
tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, adam=AdamConfig(lr))
tr.binning = "radix"
tr.step([0, 4])
tr.binning, tr.sort_cap = "bucket", 8  # large-bucket fallback path
tr.step([1, 5])
torch.cuda.synchronize()
print("radix + fallback ok", flush=True)
# bucket sort: every size class
sizes = [0, 1, 31, 32, 33, 256, 257, 511, 512, 513, 1024, 1025, 4096, 5000]
rng = np.random.default_rng(0)
total = int(sum(sizes))
depth = rng.random(total, dtype=np.float32) * 100 + 0.1
rows = rng.permutation(np.arange(total, dtype=np.uint64))
keys = (depth.view(np.uint32).astype(np.uint64) << np.uint64(32)) | rows
starts = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int32)
ranges = np.stack([starts, starts + np.asarray(sizes, dtype=np.int32)], axis=1).astype(np.int32)
kd = torch.as_tensor(keys.view(np.int64), device="cuda")
rd = torch.as_tensor(ranges.reshape(-1), device="cuda")
out = torch.empty(total, dtype=torch.int32, device="cuda")
nat.call("bs_bin_tiles_sort", nat.ptr(kd), nat.ptr(rd), len(sizes), 16384, nat.ptr(out), nat.stream_handle())
torch.cuda.synchronize()
print("bucket sorts ok", flush=True)
