"""Scheduling path of the distributed step, reference vs this framework
(SURVEY.md §8(d) CPU baseline (1)): zorder_group, build_bipartite_graph,
hierarchical_partition once; build_access_matrix + hierarchical_place +
account_iteration per batch.

    python tools/sched_timing.py --impl reference   # build container only: imports /root/reference (1 core)
    python tools/sched_timing.py --impl ours        # GPU box: this package (K0 on the GPU, native partitioner)

Both run the same workload: aerial scene (seed 5, 1M points, grid (4, 4),
128 views), G = 2048, N = 8 (topology (8, 1)), batch 16, P = 2, one epoch of
batches (schedule seed 9); the output JSON goes to stdout.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORK = dict(seed=5, n_points=1_000_000, grid=(4, 4), n_views=128, G=2048, N=8, batch=16, P=2, epochs=1)


def _api(impl):
    if impl == "reference":
        import shutil
        import tempfile

        tmp = tempfile.mkdtemp(prefix="refpkg_")
        shutil.copytree("/root/reference/pkg/src/splatsched", os.path.join(tmp, "splatsched"))
        sys.path.insert(0, tmp)
        import splatsched as api
        return api
    sys.path.insert(0, ROOT)
    import paper_2512_20017_b200 as api
    return api


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=["reference", "ours"], required=True)
    ap.add_argument("--batches", type=int, default=4, help="timed batches of the epoch")
    args = ap.parse_args()
    api = _api(args.impl)
    sync = (lambda: None)
    if args.impl == "ours":
        import torch

        sync = torch.cuda.synchronize
    w = WORK
    ds = api.generate_aerial_scene(seed=w["seed"], n_points=w["n_points"], grid=w["grid"], n_views=w["n_views"],
                                   altitude=50.0, image_size=(1920, 1080))
    out = {"impl": args.impl, "workload": dict(w, grid=list(w["grid"])), "cores": 1 if args.impl == "reference" else None}
    if args.impl == "ours":  # CUDA context, library load and kernel modules outside the timings
        small = api.generate_aerial_scene(seed=1, n_points=5000, grid=(1, 1), n_views=4, altitude=50.0)
        api.build_bipartite_graph(api.zorder_group(small.cloud, 256), small)
        sync()
    t = time.perf_counter()
    g = api.zorder_group(ds.cloud, w["G"])
    sync()
    out["zorder_group_s"] = time.perf_counter() - t
    t = time.perf_counter()
    graph = api.build_bipartite_graph(g, ds)
    sync()
    out["build_bipartite_graph_s"] = time.perf_counter() - t
    t = time.perf_counter()
    part = api.hierarchical_partition(graph, w["N"], 1, 0.05, 5)
    out["hierarchical_partition_s"] = time.perf_counter() - t
    topo = api.ClusterTopology(w["N"], 1, 25e9, 900e9)
    account_iteration = getattr(api, "account_iteration", None) or api.simulator.account_iteration
    order = np.random.default_rng(np.random.SeedSequence([9, 2, 0])).permutation(w["n_views"])
    per = {"build_access_matrix_s": [], "hierarchical_place_s": [], "account_iteration_s": []}
    inter = api.CostCoefficients(p=4.0)
    intra = api.CostCoefficients(alpha=0.0, beta=0.1, gamma=0.1, delta=1.0, p=4.0)
    for i in range(args.batches):
        batch = [ds.views[int(v)] for v in order[i * w["batch"]:(i + 1) * w["batch"]]]
        t = time.perf_counter()
        A = api.build_access_matrix(g, part, batch, w["P"])
        sync()
        per["build_access_matrix_s"].append(time.perf_counter() - t)
        t = time.perf_counter()
        sol = api.hierarchical_place(A, w["N"], 1, inter, intra)
        per["hierarchical_place_s"].append(time.perf_counter() - t)
        t = time.perf_counter()
        tr = account_iteration(A, sol, topo, 44)
        per["account_iteration_s"].append(time.perf_counter() - t)
        out.setdefault("inter_points", []).append(int(tr.send_inter.sum()))
        out.setdefault("assignment", []).append([int(x) for x in sol.assignment])
    for k, v in per.items():
        out[k] = float(np.median(v))
    out["per_batch_s"] = sum(out[k] for k in per)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
