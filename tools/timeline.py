"""Kernel timeline of one C2 training step (torch.profiler / CUPTI):
per-kernel device time and the idle gaps between consecutive kernels.

    python tools/timeline.py [--config c2] > gpurun_out/timeline.txt
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2512_20017_b200 import scenes  # noqa: E402
from paper_2512_20017_b200.trainer import AdamConfig, SplatTrainer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=1, help="consecutive steps inside the profile")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    ds, g, params, gt = bench.build_scene(cfg)[:4]
    tr = SplatTrainer(params, g.group_begin(), g.aabbs.reshape(-1, 6), ds.views, gt=gt,
                      adam=AdamConfig(scenes.lr_table(cfg["altitude"])), model=cfg.get("model", "3dgs"))
    sched = bench.schedule(cfg["n_views"], cfg["batch"], 5 + args.steps)
    for i in range(5):
        tr.step(sched[i])
    assert len(sched) >= 5 + args.steps
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for i in range(args.steps):
            tr.step(sched[5 + i])
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    prev_end = t0
    busy = 0.0
    for e in ev:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        gap = s - prev_end
        busy += d
        print(f"{(s - t0) / 1e3:8.3f} ms  gap {gap:7.1f} us  dur {d:8.1f} us  {e.name[:90]}")
        prev_end = max(prev_end, e.time_range.end)
    span = prev_end - t0
    print(f"span {span / 1e3:.3f} ms  busy {busy / 1e3:.3f} ms  idle {(span - busy) / 1e3:.3f} ms  kernels {len(ev)}")


if __name__ == "__main__":
    main()
