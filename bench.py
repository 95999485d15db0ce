"""Benchmark of the PBDR training step (BASELINE.json metric: train images/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

One process per GPU (torchrun for N > 1).  A step = forward + backward of a
batch of views + Adam (Alg. 1) on a synthetic aerial scene
of the configuration's shape (data: synthetic, random-init Gaussians).
Prints ONE JSON line on rank 0 (contract in the task statement):
  value      images/s over the timed K steps, inputs resident in HBM
  e2e        images/s through the public API with the step's ground-truth
             images copied H2D from pinned host memory and the losses read back
  roofline   dominant kernel: algorithmic bytes / CUDA-event duration vs the
             measured HBM copy bandwidth (MEASURED_PEAKS.json)
  cpu_baseline  the CPU oracle's training step on this host (bounded sample)
--impl reference times the CPU oracle alone (the reference package has no
renderer) on the host cores.

--gpus N without a torchrun environment re-launches this script under
torch.distributed.run with N local ranks (one process per GPU, NCCL; gloo
when the ranks have to share GPUs or BS_DIST_BACKEND=gloo) and relays the
rank-0 line.  Rank 0 alone builds the bipartite visibility graph and the
points-to-rank partition and broadcasts the group owners; every rank then
materialises only its own shard's Gaussian attributes.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]: 1M Gaussians, 1080p, batch 4, 1 GPU
    "c2": dict(seed=1, n_points=1_000_000, grid=(1, 1), n_views=8, altitude=50.0, image_size=(1920, 1080),
               batch=4, G=2048, desc="synthetic 3DGS aerial scene, 1M Gaussians, 1080p cameras, batch 4"),
    # configs[0]: CPU-oracle-sized case
    "c1": dict(seed=0, n_points=10_000, grid=(2, 2), n_views=8, altitude=50.0, image_size=(128, 128),
               batch=1, G=2048, desc="synthetic 3DGS scene, 10K Gaussians, 8 cameras at 128x128, batch 1"),
    # configs[2]: 2DGS (surfels), 2M points, 1080p, batch 4
    "c3": dict(seed=2, n_points=2_000_000, grid=(1, 1), n_views=8, altitude=50.0, image_size=(1920, 1080),
               batch=4, G=2048, model="2dgs",
               desc="synthetic 2DGS aerial scene, 2M surfels, 1080p cameras, batch 4"),
    # configs[3]: city scale, 50M Gaussians, 4K cameras, batch 16; strong scaling
    # over N (points sharded by the partition, the global batch stays 16);
    # ground truth only for the scheduled views (SeedSequence([seed, 5, view]));
    # selective Adam (only points visible in the batch), as the paper trains
    # its city-scale models
    "c4": dict(seed=3, n_points=50_000_000, grid=(8, 8), n_views=256, altitude=50.0, image_size=(3840, 2160),
               batch=16, G=2048, scaling="strong", gt_subset=True, selective_adam=True,
               desc="synthetic city-scale 3DGS, 50M Gaussians, 4K cameras, batch 16"),
}
METRIC = "train images/s (fwd+bwd) at 1/2/4/8 B200, % HBM roofline; comm bytes/step"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        try:
            rows = [ln.split(",") for ln in open(self.path).read().strip().splitlines() if ln.strip()]
        except Exception:
            return out
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower() == "active":
                    reasons.add(nm)
        if sm:
            out.update(sm_mhz=statistics.median(sm), sm_max_mhz=max(smax), reasons=sorted(reasons), samples=len(sm))
        return out


def build_scene(cfg, gt_views=None, world=1, rank=0):
    """Scene, Z-order groups, this rank's Gaussian attributes and ground truth
    (all views, or only `gt_views` when the configuration asks for a subset).
    N = 1: every point.  N > 1: the shard of `shard_for_rank` only (the
    attribute stream is drawn in blocks and only the shard's rows are kept).
    Returns ds, g, params, gt, group_begin, aabb, partition info."""
    from paper_2512_20017_b200 import scenes
    from paper_2512_20017_b200.culling import zorder_group

    ds = scenes.generate_aerial_scene(cfg["seed"], cfg["n_points"], cfg["grid"], cfg["n_views"], cfg["altitude"],
                                      cfg["image_size"])
    g = zorder_group(ds.cloud, G=cfg["G"])
    spacing = scenes.mean_spacing(cfg["altitude"], cfg["grid"], cfg["n_points"])
    info = {}
    if world > 1:
        rows, gb, aabb, info = shard_for_rank(ds, g, world, rank)
        params = scenes.init_gaussians_rows(g.sorted_cloud, cfg["seed"], spacing, rows)
        info["rows"] = rows
    else:
        params = scenes.init_gaussians(g.sorted_cloud, cfg["seed"], spacing)
        gb, aabb = g.group_begin(), g.aabbs.reshape(-1, 6)
    W, H = cfg["image_size"]
    if cfg.get("gt_subset") and gt_views is not None:
        gt = scenes.synthetic_gt_views(cfg["seed"], gt_views, W, H)
    else:
        gt = scenes.synthetic_gt(cfg["seed"], cfg["n_views"], W, H)
    return ds, g, params, gt, gb, aabb, info


def schedule(n_views, batch, steps, seed=9):
    """Batches as in run_training_sim (simulator.py:350-358): per epoch a
    SeedSequence([seed, 2, e]) permutation of the views, partial batch dropped."""
    out, e = [], 0
    while len(out) < steps:
        order = np.random.default_rng(np.random.SeedSequence([seed, 2, e])).permutation(n_views)
        for i in range(n_views // batch):
            out.append([int(v) for v in order[i * batch:(i + 1) * batch]])
        e += 1
    return out[:steps]


def weak_scaled(cfg, world):
    """N ranks: N aerial cells side by side (grid (1, N)), N x the points,
    views and batch -- per-rank work fixed (weak scaling)."""
    c = dict(cfg)
    rows, cols = cfg["grid"]
    c.update(n_points=cfg["n_points"] * world, grid=(rows, cols * world), n_views=cfg["n_views"] * world,
             desc=cfg["desc"] + f" per rank, x{world} ranks (grid {rows}x{cols * world})")
    return c


def shard_for_rank(ds, g, world, rank):
    """Points-to-rank map of the paper's offline placement: GPU-built
    bipartite visibility graph -> hierarchical_partition(graph, N, 1), run by
    rank 0 alone and broadcast as the per-group owner (every rank needs all
    owners: the random baseline and the comm report replay them).  Returns
    this rank's point rows (ascending global index, whole groups), its group
    table and AABBs, and the partition info."""
    import torch
    import torch.distributed as dist

    from paper_2512_20017_b200.sharding import build_bipartite_graph, hierarchical_partition

    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    owner_t = torch.empty(g.n_groups, dtype=torch.int64, device=dev)
    stats = torch.zeros(4, dtype=torch.float64, device=dev)
    if rank == 0:
        t0 = time.time()
        graph = build_bipartite_graph(g, ds)
        t1 = time.time()
        part = hierarchical_partition(graph, world, 1, eps=0.05, seed=5)
        t2 = time.time()
        owner_t.copy_(torch.as_tensor(np.asarray(part.flat_gpus(), dtype=np.int64)))
        stats.copy_(torch.tensor([len(graph.edge_weights), t1 - t0, t2 - t1, 0.0], dtype=torch.float64))
    dist.broadcast(owner_t, 0)
    dist.broadcast(stats, 0)
    owner = owner_t.cpu().numpy()
    gbeg = g.group_begin().astype(np.int64)
    sizes_all = np.diff(gbeg)
    mine = np.flatnonzero(owner == rank)
    sizes = sizes_all[mine]
    rows = np.concatenate([np.arange(gbeg[k], gbeg[k + 1]) for k in mine]) if len(mine) else np.zeros(0, np.int64)
    gb = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    aabb = g.aabbs.reshape(-1, 6)[mine]
    per_rank = np.bincount(owner, weights=sizes_all, minlength=world).astype(np.int64)
    e, tg, tp = stats.cpu().tolist()[:3]
    info = {"groups": int(g.n_groups), "graph_edges": int(e), "graph_build_s": round(tg, 2),
            "partition_s": round(tp, 2), "points_per_rank": [int(x) for x in per_rank], "built_on": "rank 0",
            "owner": owner}
    return rows, gb, aabb, info


def comm_bytes_report(comm, step_AW, batches, ds, g, world, rank, steps, row_bytes=48, grad_bytes=36, P=1):
    """All-to-all bytes per step: moved by NCCL (summed over ranks),
    A-predicted (account_iteration on topology (N, 1)), and the same
    accounting for the RandomStrategy baseline on the same batches."""
    import torch

    from paper_2512_20017_b200.accounting import (ClusterTopology, account_iteration, random_placement,
                                                  random_point_gpus)
    from paper_2512_20017_b200.culling import build_access_matrix

    dev = "cpu" if comm.host_staging else "cuda"
    t = torch.tensor([comm.bytes_fwd, comm.bytes_bwd], dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(t)
    fwd, bwd = (float(x) / steps for x in t.tolist())
    topo = ClusterTopology(world, 1, 25e9, 300e9)
    pred = np.mean([account_iteration(A, __import__("paper_2512_20017_b200").PlacementSolution(W, world), topo,
                                      row_bytes).send_inter.sum() for A, W in step_AW]) * row_bytes
    rnd_pg = random_point_gpus(len(ds.cloud), world,
                               np.random.default_rng(np.random.SeedSequence([5, 17])))[g.permutation]
    rnd = []
    for it, b in enumerate(batches):
        A = build_access_matrix(g, rnd_pg, [ds.views[v] for v in b], P)
        sol = random_placement(len(b) * P * P, world, np.random.default_rng(np.random.SeedSequence([5, 3, it])))
        rnd.append(account_iteration(A, sol, topo, row_bytes).send_inter.sum() * row_bytes)
    rnd = float(np.mean(rnd))
    return {"fwd_bytes_per_step": fwd, "bwd_bytes_per_step": bwd, "fwd_bytes_predicted": float(pred),
            "random_fwd_bytes_per_step": rnd, "reduction_vs_random_pct": 100.0 * (1.0 - fwd / rnd) if rnd else None,
            "row_bytes": {"fwd": row_bytes, "bwd": grad_bytes}, "patches_per_side": P,
            "note": "moved = render sets (P > 1 adds splats crossing patch borders); predicted/random = access "
                    "matrix (account_iteration, topology (N, 1)); forward bytes per row = splat state + 4-byte id"}


_STAGE_KERNEL = {"raster_bwd": "raster_bwd_kernel", "raster_fwd": "raster_fwd_kernel", "raster": "raster_fused_kernel", "raster2d": "raster2d_fused_kernel",
                 "raster2d_bwd": "raster2d_bwd_kernel", "raster2d_fwd": "raster2d_fwd_kernel",
                 "project_bwd_adam": "project_bwd_adam_kernel", "project": "project_fwd_kernel", "cull": "cull_kernel"}

# committed ncu --set full summaries (newest first) per (model, configuration)
# they captured (per launch of that workload: counts and bytes do not transfer)
TRAFFIC_FILES = {("3dgs", "c2"): ("r2z_kernel_traffic.json", "r2u_kernel_traffic.json", "r2v_kernel_traffic.json", "r2y_kernel_traffic.json", "r2g_kernel_traffic.json",
                                  "r2_kernel_traffic.json", "r1_kernel_traffic.json"),
                 ("2dgs", "c3"): ("r2z_kernel_traffic.json", "r2u_kernel_traffic.json", "r2v_kernel_traffic.json", "r2y_kernel_traffic.json", "r2g_kernel_traffic.json",
                                  "r2_kernel_traffic.json", "r1_kernel_traffic.json"),
                 ("3dgs", "c4"): ("r2v_kernel_traffic_c4.json", "r2y_kernel_traffic_c4.json")}
_PROFILED = {"3dgs": "c2", "2dgs": "c3"}


def kernel_profile(stage, model="3dgs", config=None):
    """Entry of the newest committed ncu --set full summary (profiles/) for
    one launch of the stage's kernel, or {} when no capture of this
    configuration is committed (counts and bytes are per launch of that workload)."""
    files = TRAFFIC_FILES.get((model, config if config is not None else _PROFILED.get(model)), ())
    for name in files:
        try:
            table = json.load(open(os.path.join(ROOT, "profiles", name)))
        except Exception:
            continue
        key = stage.replace("raster_", "raster2d_") if model == "2dgs" and stage.startswith("raster_") else stage
        if model == "2dgs" and stage == "raster":
            key = "raster2d"
        prefix = _STAGE_KERNEL.get(key, key)
        model_tag = "Model2" if model == "2dgs" else "Model3"
        hits = [v for k, v in table.items() if k.startswith(prefix)]
        tagged = [v for k, v in table.items() if k.startswith(prefix) and model_tag in k]
        ent = (tagged or hits or [{}])[0]
        if ent:
            return dict(ent, source=f"profiles/{name}")
    return {}


def _max_over_ranks(vals):
    import torch
    import torch.distributed as dist

    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def dist_backend(world: int) -> str:
    """NCCL when every rank has its own GPU; gloo (host-staged exchanges) when
    ranks have to share GPUs (NCCL refuses two ranks on one device) or when
    BS_DIST_BACKEND says so."""
    import torch

    forced = os.environ.get("BS_DIST_BACKEND")
    if forced:
        return forced
    return "nccl" if torch.cuda.device_count() >= world else "gloo"


def config_dict(cfg, B, world, P):
    """The `config` of the JSON line, identical in both arms."""
    return {"workload": cfg["desc"], "primitive": cfg.get("model", "3dgs"), "n_points": cfg["n_points"],
            "optimizer": "selective Adam" if cfg.get("selective_adam") else "Adam",
            "image": list(cfg["image_size"]), "global_batch": B, "views": cfg["n_views"], "group_size": cfg["G"],
            "parallelism": f"points+images x{world}", "patches_per_side": P,
            "l2": "inputs larger than L2 (params + Adam state %.0f MB over the scene; L2 126 MB)"
                  % (cfg["n_points"] * 720 / 1e6)}


def run_ours(args, cfg):
    import torch

    from paper_2512_20017_b200 import _native as nat
    from paper_2512_20017_b200 import scenes
    from paper_2512_20017_b200.trainer import AdamConfig, SplatTrainer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    comm, part_info, backend = None, {}, None
    if world > 1:
        import torch.distributed as dist

        from paper_2512_20017_b200.exchange import PeerExchange, SplatExchange

        backend = dist_backend(world)
        dist.init_process_group(backend)
        if cfg.get("scaling", "weak") == "weak":
            cfg = weak_scaled(cfg, world)
    strong = cfg.get("scaling", "weak") == "strong"
    B = cfg["batch"] if strong else cfg["batch"] * world
    sched = schedule(cfg["n_views"], B, args.warmup + 2 * args.steps + 2)
    gt_ids = sorted({v for b in sched for v in b}) if cfg.get("gt_subset") else None
    t0 = time.time()
    ds, g, params, gt, gb, aabb, part_info = build_scene(cfg, gt_views=gt_ids, world=world, rank=rank)
    gt_row = (lambda v: v) if gt_ids is None else {v: k for k, v in enumerate(gt_ids)}.__getitem__
    if world > 1:
        # peer: the splat rows / gradients move by loads and stores into the
        # renderers' / owners' memory (CUDA IPC over NVLink, fused into the
        # projection and the gradient return); collective: torch.distributed
        # all_to_all_single (NCCL; host-staged over gloo)
        comm = PeerExchange.create() if args.exchange == "peer" else SplatExchange()
    setup_s = time.time() - t0
    W, H = cfg["image_size"]
    model = cfg.get("model", "3dgs")
    P = args.patches or cfg.get("P", 1)
    tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt,
                      adam=AdamConfig(scenes.lr_table(cfg["altitude"]), selective=bool(cfg.get("selective_adam"))),
                      comm=comm, model=model, gt_view_ids=gt_ids, patches=P, global_ids=part_info.get("rows"))
    # clocks are sampled from the start of the warm-up to the end of the timed
    # region (nvidia-smi needs ~0.5 s to start streaming)
    clk = ClockSampler(local).__enter__()
    time.sleep(1.0)
    nxt = (lambda i: sched[i + 1]) if comm is not None else (lambda i: None)  # async placement (N > 1)
    for i in range(args.warmup):
        tr.step(sched[i], next_batch=nxt(i))
    torch.cuda.synchronize()
    # ---- timed region: device-resident inputs
    tr.timers = {}
    lc0 = nat.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    inst, rows, big = [], [], []
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    step_AW = []
    if comm is not None:
        comm.bytes_fwd = comm.bytes_bwd = 0
    # no Python garbage collection inside the timed loops: a collection pass
    # stalls the host between two launches and leaves the GPU idle
    gc.collect()
    gc.disable()
    start.record()
    if comm is not None:
        comm.place_ms.clear()
        comm.wait_ms.clear()
    for i in range(args.steps):
        tr.step(sched[args.warmup + i], next_batch=nxt(args.warmup + i))
        inst.append(tr.last["n_inst"])
        rows.append(tr.last["n_rows"])
        big.append(int(tr.last.get("largest_bucket", 0)))
        if comm is not None:
            step_AW.append((tr.last["A"], tr.last["W"]))
    end.record()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk.__exit__(None, None, None)
    gc.enable()
    launches = nat.launch_count() - lc0
    tr.last["n_visible_points"] = int((tr.buf.bufs["mask"][: tr.S] != 0).sum().item())
    ms = start.elapsed_time(end)
    if world > 1:
        ms = _max_over_ranks([ms])[0]
    stage_ms = {k: float(np.mean([s.elapsed_time(e) for s, e in v])) for k, v in tr.timers.items()}
    tr.timers = None
    ms_per_step = ms / args.steps
    images = B * args.steps
    value = images / (ms / 1000.0)
    comm_report = None
    placement = None
    if comm is not None:
        placement = {"async": True, "stale_steps": 1, "host_place_ms": round(float(np.mean(comm.place_ms)), 3),
                     "step_wait_ms": round(float(np.mean(comm.wait_ms)), 3) if comm.wait_ms else None}
        # forward rows travel with their point's 4-byte global id (canonical order)
        comm_report = comm_bytes_report(comm, step_AW, sched[args.warmup:args.warmup + args.steps], ds, g,
                                        world, rank, args.steps, row_bytes=4 * (tr.sp_floats + 1),
                                        grad_bytes=4 * tr.gsp_wire_floats, P=P)
        peer = getattr(comm, "peer", False) and P == 1
        comm_report.update(backend=backend, communicator_size=world,
                           exchange="peer memory (CUDA IPC: rows written by the projection / gradient return "
                                    "into the destination's buffer, stream-ordered flags)" if peer
                           else "torch.distributed all_to_all_single",
                           collectives_per_step={"all_gather": 1, "all_to_all_single": 0 if peer else
                                                 (2 if P == 1 else 3)})
    # ---- e2e: public API with pinned host ground truth, loss read back
    # the step's ground-truth images are copied from pinned host memory on a
    # side stream, double-buffered: step i+1's upload overlaps step i
    pinned = torch.from_numpy(gt).pin_memory()
    # the same batches as the device-timed region, so that e2e and `value`
    # measure the same work (per-step cost depends on which views a batch holds)
    e2e_sched = sched[args.warmup: args.warmup + args.steps]
    gt_bufs = [torch.empty((B, H, W, 3), dtype=torch.uint8, device="cuda") for _ in range(2)]
    copy_stream = torch.cuda.Stream()

    def e2e_run(batches):
        """The step loop a user runs: per step the batch's ground truth goes
        H2D (side stream, double-buffered: step i+1's upload overlaps step i)
        and the losses come back D2H into pinned memory.  Returns (device ms,
        wall ms, last losses)."""
        ready, freed = [None, None], [None, None]

        def upload(i):
            with torch.cuda.stream(copy_stream):
                if freed[i % 2] is not None:
                    copy_stream.wait_event(freed[i % 2])
                for k, v in enumerate(batches[i]):
                    gt_bufs[i % 2][k].copy_(pinned[gt_row(v)], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_stream)
                ready[i % 2] = ev

        # per-step losses land in pinned host memory by an asynchronous D2H
        # copy (read back every step without stalling the launch queue)
        loss_pinned = [torch.empty(B, dtype=torch.float32, pin_memory=True) for _ in range(len(batches))]
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_start.record()
        upload(0)
        for i, b in enumerate(batches):
            # the step waits for its upload only at the first read of the
            # ground truth (the raster): culling, projection and binning overlap it
            losses = tr.step(b, gt_batch=gt_bufs[i % 2], gt_ready=ready[i % 2],
                             next_batch=batches[i + 1] if comm is not None and i + 1 < len(batches) else None)
            ev = torch.cuda.Event()
            ev.record()
            freed[i % 2] = ev
            if i + 1 < len(batches):
                # queued once the host is back from step i (which returns while
                # its raster runs): the next upload overlaps the compute-bound
                # raster rather than the memory-bound front of the step
                upload(i + 1)
            loss_pinned[i][: losses.numel()].copy_(losses, non_blocking=True)
        e_end.record()
        torch.cuda.synchronize()
        return e_start.elapsed_time(e_end), (time.perf_counter() - t0) * 1000.0, loss_pinned[-1]

    e2e_run(sched[:max(1, min(args.warmup, 3))])  # warm-up of the e2e path (untimed)
    gc.collect()
    gc.disable()
    e2e_ms, e2e_wall, loss_host = e2e_run(e2e_sched)
    gc.enable()
    if world > 1:
        e2e_ms, e2e_wall = _max_over_ranks([e2e_ms, e2e_wall])
    e2e_value = B * len(e2e_sched) / (max(e2e_ms, e2e_wall) / 1000.0)
    # ---- rooflines (paper_2512_20017_b200/roofline.py): every stage's
    # compulsory bytes vs the measured HBM peak, the step's total, and the
    # issue rate of the kernels ncu captured
    from paper_2512_20017_b200 import roofline as rl

    peak, peak_kind = rl.peaks(ROOT)
    clk_summary = clk.summary()
    counts = {"S": tr.S, "V": int(np.mean(rows)), "Vp": int(tr.last.get("n_visible_points", tr.S)),
              "I": int(np.mean(inst)), "Np": int(tr.last["n_slots"]) * H * W,
              "nb": int(tr.last["n_slots"]) * tr.tiles,
              "gsp_clear": comm is None and model == "3dgs" and tr.binning != "radix",
              "selective": bool(tr.adam.selective)}
    stages = {}
    for k, v in stage_ms.items():
        nb = rl.stage_bytes(k, counts, model)
        h = rl.hbm(nb, v, peak) if nb else None
        prof = kernel_profile(k, model, args.config)
        iss = rl.issue(prof.get("warp_instructions"), v, clk_summary.get("sm_mhz"))
        stages[k] = {"ms": round(v, 4), "share": round(v / ms_per_step, 4),
                     "gbs": round(h["achieved"], 1) if h else None, "hbm_frac": round(h["frac"], 4) if h else None,
                     "issue_frac": iss["frac"] if iss else None, "binding": rl.binding(h, iss)}
    dom = max(stage_ms, key=stage_ms.get) if stage_ms else None
    roof = None
    if dom:
        nbytes = rl.stage_bytes(dom, counts, model)
        h = rl.hbm(nbytes, stage_ms[dom], peak)
        prof = kernel_profile(dom, model, args.config)
        iss = rl.issue(prof.get("warp_instructions"), stage_ms[dom], clk_summary.get("sm_mhz"))
        sb = rl.step_bytes(counts, model, stages=tuple(stage_ms))
        roof = {"kernel": dom, "bound": "hbm", "achieved": h["achieved"], "peak": peak, "unit": "GB/s",
                "frac": h["frac"], "traffic": prof.get("dram_traffic_bytes"), "peak_kind": peak_kind,
                "bytes_per_launch": nbytes, "ms_per_launch": stage_ms[dom],
                "binding": rl.binding(h, iss), "issue": iss,
                "traffic_source": prof.get("source"),
                "step_hbm": {"bytes_per_step": sb, "achieved": round(sb / (ms_per_step / 1000.0) / 1e9, 1),
                             "peak": peak, "frac": round(sb / (ms_per_step / 1000.0) / 1e9 / peak, 4),
                             "survey_formula_bytes": rl.survey_step_bytes(counts)},
                "note": "bound/achieved/frac: the contract's HBM roofline of the dominant kernel (algorithmic bytes "
                        "of roofline.py / CUDA-event launch time); binding: the bound it actually sits at "
                        "(issue = executed warp instructions of the same launch in the committed ncu capture / "
                        "launch time vs 148 SMs x 4 schedulers x the sampled SM clock); step_hbm: compulsory "
                        "bytes of every stage of the step / ms_per_step"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, ds, g, params, gt, steps=1, gt_row=gt_row)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(cfg, B, world, P),
            "e2e": {"value": round(e2e_value, 3), "unit": "images/s", "device_ms": round(e2e_ms, 3),
                    "wall_ms": round(e2e_wall, 3), "h2d_bytes_per_step": B * H * W * 3 * world,
                    "d2h_bytes_per_step": 4 * B},
            "comm": comm_report,
            "placement": placement,
            "partition": {k: v for k, v in part_info.items() if k not in ("owner", "rows")} or None,
            "roofline": roof,
            "stages": stages,
            "instances_per_step": int(np.mean(inst)), "splat_rows_per_step": int(np.mean(rows)),
            "largest_tile_bucket": int(max(big)) if big else None,
            "gpu_launches": int(launches),
            "clocks": clk_summary,
            "cpu_baseline": cpu,
            "setup_s": round(setup_s, 1),
            "final_loss": None if loss_host is None else [round(float(x), 5) for x in loss_host],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        if hasattr(comm, "close"):
            comm.close()
        torch.distributed.destroy_process_group()


def cpu_baseline(cfg, ds, g, params, gt, steps=1, warmup=0, gt_row=lambda v: v):
    """CPU oracle training step on this host, bounded sample: 1 view of the
    configuration per step, all host threads."""
    from oracle import py_oracle
    from paper_2512_20017_b200 import scenes
    from paper_2512_20017_b200.culling import batch_planes
    from paper_2512_20017_b200.trainer import camera_bytes

    p = np.ascontiguousarray(params.copy())
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    lr = scenes.lr_table(cfg["altitude"])
    model = cfg.get("model", "3dgs")
    views = [ds.views[i % len(ds.views)] for i in range(steps + warmup)]
    for k in range(warmup):
        py_oracle.train_step(p, m, v, batch_planes([views[k]], 1), camera_bytes([views[k]]),
                             gt[gt_row(views[k].id):gt_row(views[k].id) + 1], 3, lr, 0.9, 0.999, 1e-15, k + 1,
                             model=model)
    t0 = time.perf_counter()
    for k in range(warmup, warmup + steps):
        vv = views[k]
        py_oracle.train_step(p, m, v, batch_planes([vv], 1), camera_bytes([vv]), gt[gt_row(vv.id):gt_row(vv.id) + 1], 3,
                             lr, 0.9,
                             0.999, 1e-15, k + 1, model=model)
    dt = time.perf_counter() - t0
    return {"value": round(steps / dt, 5), "unit": "images/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"{steps} step(s) x 1 view of the same scene ({cfg['n_points']} Gaussians, "
                      f"{cfg['image_size'][0]}x{cfg['image_size'][1]}), oracle/splat_oracle.c OpenMP",
            "seconds": round(dt, 2)}


def run_reference(args, cfg):
    """The reference arm: the CPU implementation of the path (the oracle port,
    oracle/splat_oracle.c; the reference package itself has no renderer,
    SURVEY.md §0) on all host cores, rank 0 only.  Each step is a bounded
    sample of the workload -- ONE view of the configuration's scene through
    the full training step (cull, project, bin, blend, L1, backward, Adam) --
    so images/s compares per image with the GPU arm's batches."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and cfg.get("scaling", "weak") == "weak":
        cfg = weak_scaled(cfg, world)
    strong = cfg.get("scaling", "weak") == "strong"
    B = cfg["batch"] if strong else cfg["batch"] * world
    P = args.patches or cfg.get("P", 1)
    ds, g, params, gt, gt_row = build_scene_host(cfg, args.steps + min(args.warmup, 1))
    cpu = cpu_baseline(cfg, ds, g, params, gt, steps=args.steps, warmup=min(args.warmup, 1), gt_row=gt_row)
    line = {"metric": METRIC, "impl": "reference", "value": cpu["value"], "unit": "images/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000.0 / cpu["value"], 2), "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(cfg, B, world, P),
            "cpu_baseline": cpu,
            "e2e": {"value": cpu["value"], "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "each reference step is 1 view of the configuration's scene (bounded CPU sample); "
                    "images/s is per image, like the GPU arm's"}
    print(json.dumps(line), flush=True)


def build_scene_host(cfg, n_used=None):
    """Scene on the host only (reference arm: no GPU involvement)."""
    from oracle import py_oracle
    from paper_2512_20017_b200 import scenes

    ds = scenes.generate_aerial_scene(cfg["seed"], cfg["n_points"], cfg["grid"], cfg["n_views"], cfg["altitude"],
                                      cfg["image_size"])
    perm, gb, aabb = py_oracle.zorder_layout(ds.cloud.positions, cfg["G"])
    sorted_cloud = scenes.PointCloud(ds.cloud.positions[perm])
    params = scenes.init_gaussians(sorted_cloud, cfg["seed"],
                                   scenes.mean_spacing(cfg["altitude"], cfg["grid"], cfg["n_points"]))
    W, H = cfg["image_size"]
    if cfg.get("gt_subset") and n_used is not None:
        ids = [i % cfg["n_views"] for i in range(n_used)]
        return (ds, None, params, scenes.synthetic_gt_views(cfg["seed"], ids, W, H),
                {v: k for k, v in enumerate(ids)}.__getitem__)
    return ds, None, params, scenes.synthetic_gt(cfg["seed"], cfg["n_views"], W, H), (lambda v: v)


def spawn(args) -> int:
    """--gpus N outside torchrun: re-launch this script as N local ranks
    (torch.distributed.run, rendezvous on 127.0.0.1); rank 0 prints the line."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--patches", type=int, default=0, help="patches per image side P (default: the config's, 1)")
    ap.add_argument("--exchange", default="peer", choices=["peer", "collective"],
                    help="N > 1: splat-row exchange through peer memory (default) or torch.distributed all-to-alls")
    args = ap.parse_args()
    world = os.environ.get("WORLD_SIZE")
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if world is None and args.gpus > 1:
        sys.exit(spawn(args))
    if world is not None and int(world) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
