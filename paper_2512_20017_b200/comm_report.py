"""All-to-all bytes per step, locality-aware vs random partitioning, at the
BASELINE multi-GPU configurations (configs[3] C4 and configs[4] C5).

    python -m paper_2512_20017_b200.comm_report --config c4 --gpus 2 4 8 [--epochs 1] [--out FILE]

For every N the reference's own experiment (simulator.py:293-413 ->
accounting.run_training_sim) is run on the synthetic scene of the
configuration with ClusterTopology(N, 1) -- on one NVSwitch box every GPU is
its own "machine", so forward inter-machine points are exactly the points
the SP all-to-all moves -- once with the paper's
LocalityAwareStrategy (GPU-built bipartite graph, native multilevel
partitioner, per-step hierarchical_place) and once with RandomStrategy, on
the same batch schedule.  Bytes are reported for the reference's accounting
unit (profile bytes per point, 44 B) and for the rows this framework's
exchange actually moves (SP 48 B + the point's 4-byte global id forward,
G_SP 36 B backward).  The access
matrices come from the sm_100a culling kernel; no training step runs.
"""

from __future__ import annotations

import argparse
import json
import os
import time

import numpy as np

from . import scenes
from .accounting import (ClusterTopology, LocalityAwareStrategy, RandomStrategy, comm_reduction,
                         run_training_sim)
from .assign import CostCoefficients

# scene calls, batch, patch factor and seeds of the configs
CONFIGS = {
    "c4": dict(seed=3, n_points=50_000_000, grid=(8, 8), n_views=256, image_size=(3840, 2160), batch=16, P=1,
               G=2048, desc="synthetic city-scale 3DGS, 50M Gaussians, 4K cameras, batch 16"),
    "c5": dict(seed=4, n_points=200_000_000, grid=(16, 16), n_views=1024, image_size=(1920, 1080), batch=32, P=2,
               G=2048, desc="200M-point aerial synthetic scene, batch 32, 1080p, P=2"),
    # small smoke configuration (tests)
    "tiny": dict(seed=0, n_points=200_000, grid=(4, 4), n_views=32, image_size=(640, 360), batch=8, P=1, G=2048,
                 desc="200k-point aerial scene, batch 8"),
}
SP_BYTES, GSP_BYTES = 48 + 4, 36  # forward rows travel with their global id (canonical order)


def run(cfg: dict, gpus, epochs: int = 1, log=print) -> dict:
    t0 = time.perf_counter()
    ds = scenes.generate_aerial_scene(cfg["seed"], cfg["n_points"], cfg["grid"], cfg["n_views"], 50.0,
                                      cfg["image_size"])
    t_scene = time.perf_counter() - t0
    out = {"workload": cfg["desc"], "n_points": cfg["n_points"], "views": cfg["n_views"], "batch": cfg["batch"],
           "P": cfg["P"], "group_size": cfg["G"], "epochs": epochs, "scene_s": round(t_scene, 1),
           "profile_bytes_per_point": ds.profile.bytes_per_point, "per_gpus": {}}
    inter = CostCoefficients(p=4.0)
    intra = CostCoefficients(alpha=0.0, beta=0.1, gamma=0.1, delta=1.0, p=4.0)
    for N in gpus:
        topo = ClusterTopology(N, 1, 25e9, 900e9)
        t1 = time.perf_counter()
        ours = run_training_sim(ds, topo, LocalityAwareStrategy(cfg["G"], 0.05, 5, inter, intra), epochs,
                                cfg["batch"], cfg["P"], seed=9)
        t2 = time.perf_counter()
        base = run_training_sim(ds, topo, RandomStrategy(seed=5), epochs, cfg["batch"], cfg["P"], seed=9)
        t3 = time.perf_counter()
        steps = len(ours.traces)
        pts_ours = ours.total_inter_points_forward / steps
        pts_rand = base.total_inter_points_forward / steps
        comp = np.array([t.comp for t in ours.traces], dtype=np.float64)
        row = {
            "steps": steps,
            "fwd_points_per_step": {"locality": pts_ours, "random": pts_rand},
            "reduction_pct": comm_reduction(base, ours),
            "fwd_bytes_per_step": {"locality": pts_ours * SP_BYTES, "random": pts_rand * SP_BYTES},
            "bwd_bytes_per_step": {"locality": pts_ours * GSP_BYTES, "random": pts_rand * GSP_BYTES},
            "profile_bytes_per_step": {"locality": pts_ours * ds.profile.bytes_per_point,
                                       "random": pts_rand * ds.profile.bytes_per_point},
            "rendered_points_per_step": float(comp.sum(axis=1).mean()),
            "max_rank_rendered_points_per_step": float(comp.max(axis=1).mean()),
            "locality_sim_s": round(t2 - t1, 1),
            "random_sim_s": round(t3 - t2, 1),
        }
        out["per_gpus"][str(N)] = row
        log(f"[comm_report] N={N}: {json.dumps(row)}")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--gpus", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--epochs", type=int, default=1)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    res = run(cfg, args.gpus, args.epochs)
    res["config"] = args.config
    text = json.dumps(res, indent=1)
    if args.out:
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        with open(args.out, "w") as f:
            f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
