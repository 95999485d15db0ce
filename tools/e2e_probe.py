import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import bench
from paper_2512_20017_b200 import scenes
from paper_2512_20017_b200.trainer import AdamConfig, SplatTrainer
cfg = bench.CONFIGS["c2"]
ds, g, params, gt = bench.build_scene(cfg)
tr = SplatTrainer(params, g.group_begin(), g.aabbs.reshape(-1, 6), ds.views, gt=gt, adam=AdamConfig(scenes.lr_table(cfg["altitude"])))
B = cfg["batch"]; H, W = tr.H, tr.W
sched = bench.schedule(cfg["n_views"], B, 40)
for i in range(3): tr.step(sched[i])
torch.cuda.synchronize()
def timed(fn, n=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for i in range(n): fn(i)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
print("plain", timed(lambda i: tr.step(sched[3 + i])))
print("plain again", timed(lambda i: tr.step(sched[3 + i])))
gtb = torch.as_tensor(gt[:B]).cuda()
print("gt_batch resident", timed(lambda i: tr.step(sched[3 + i], gt_batch=gtb)))
pinned = torch.from_numpy(gt).pin_memory()
def up(i):
    for k, v in enumerate(sched[3 + i]): gtb[k].copy_(pinned[v], non_blocking=True)
    tr.step(sched[3 + i], gt_batch=gtb)
print("gt_batch H2D same stream", timed(up))
lp = torch.empty(B, dtype=torch.float32, pin_memory=True)
def up2(i):
    l = tr.step(sched[3 + i]); lp.copy_(l, non_blocking=True)
print("plain + loss D2H", timed(up2))
tr.timers = {}
print("plain + stage timers", timed(lambda i: tr.step(sched[3 + i])))
tr.timers = None
bufs = [torch.empty((B, H, W, 3), dtype=torch.uint8, device="cuda") for _ in range(2)]
cs = torch.cuda.Stream()
ready, freed = [None, None], [None, None]
def upload(i):
    with torch.cuda.stream(cs):
        if freed[i % 2] is not None:
            cs.wait_event(freed[i % 2])
        for k, v in enumerate(sched[3 + i]):
            bufs[i % 2][k].copy_(pinned[v], non_blocking=True)
        ev = torch.cuda.Event(); ev.record(cs); ready[i % 2] = ev
def e2e(i):
    if i == 0: upload(0)
    upload(i + 1)
    torch.cuda.current_stream().wait_event(ready[i % 2])
    l = tr.step(sched[3 + i], gt_batch=bufs[i % 2])
    ev = torch.cuda.Event(); ev.record(); freed[i % 2] = ev
    lp.copy_(l, non_blocking=True)
print("bench-style e2e", timed(e2e))
freed = [None, None]
def e2e_nowait(i):
    if i == 0: upload(0)
    upload(i + 1)
    l = tr.step(sched[3 + i], gt_batch=bufs[i % 2])
    lp.copy_(l, non_blocking=True)
print("side-stream copies, no waits (overlap only)", timed(e2e_nowait))
