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
    ap.add_argument("--e2e", action="store_true",
                    help="bench.py's e2e loop: ground truth H2D on a side stream (double-buffered), losses D2H")
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
    W, H = cfg["image_size"]
    B = cfg["batch"]
    pinned = torch.from_numpy(gt).pin_memory()
    gt_bufs = [torch.empty((B, H, W, 3), dtype=torch.uint8, device="cuda") for _ in range(2)]
    copy_stream = torch.cuda.Stream()
    ready, freed = [None, None], [None, None]
    batches = sched[5:5 + args.steps]

    def upload(i):
        with torch.cuda.stream(copy_stream):
            if freed[i % 2] is not None:
                copy_stream.wait_event(freed[i % 2])
            for k, v in enumerate(batches[i]):
                gt_bufs[i % 2][k].copy_(pinned[v], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
            ready[i % 2] = ev

    loss_pinned = torch.empty(B, dtype=torch.float32, pin_memory=True)
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        if args.e2e:
            upload(0)
        for i in range(args.steps):
            if not args.e2e:
                tr.step(batches[i])
                continue
            losses = tr.step(batches[i], gt_batch=gt_bufs[i % 2], gt_ready=ready[i % 2])
            ev = torch.cuda.Event()
            ev.record()
            freed[i % 2] = ev
            if i + 1 < args.steps:
                upload(i + 1)
            loss_pinned.copy_(losses, non_blocking=True)
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
