"""Generate golden vectors from the UNMODIFIED reference package.

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden.py
It imports splatsched from a scratch copy of /root/reference/pkg/src and
writes small .npz/.json fixtures next to this script.  Those fixtures travel
with the repo; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"


def _import_reference():
    tmp = tempfile.mkdtemp(prefix="refpkg_")
    shutil.copytree(os.path.join(REF, "splatsched"), os.path.join(tmp, "splatsched"))
    sys.path.insert(0, tmp)
    import splatsched  # noqa: F401

    return tmp


def main():
    _import_reference()
    import splatsched as ss
    from splatsched import partition as spart
    from splatsched import placement as splace
    from splatsched import simulator as ssim
    from splatsched import visibility as svis

    out = {}

    # ---- Morton codes (visibility.py:33-62) -------------------------------
    rng = np.random.default_rng(11)
    pts = rng.uniform(-3, 7, (500, 3)).astype(np.float32)
    bbox = np.stack([pts.min(0), pts.max(0)])
    for bits in (1, 4, 10, 21):
        out[f"morton_pts"] = pts
        out[f"morton_bbox"] = bbox
        out[f"morton_codes_b{bits}"] = svis.morton_codes(pts, bbox, bits)
    # degenerate extent axis
    flat = pts.copy()
    flat[:, 2] = 1.25
    out["morton_flat_pts"] = flat
    out["morton_flat_codes"] = svis.morton_codes(flat, np.stack([flat.min(0), flat.max(0)]), 21)

    # ---- scenes + zorder (scene.py:282-462, visibility.py:113-134) ---------
    ds = ss.generate_aerial_scene(seed=3, n_points=6000, grid=(2, 3), n_views=10, altitude=20,
                                  image_size=(96, 64))
    out["aerial_positions"] = ds.cloud.positions
    out["aerial_cam_pos"] = np.stack([v.position for v in ds.views])
    out["aerial_cam_rot"] = np.stack([v.rotation for v in ds.views])
    g = ss.zorder_group(ds.cloud, G=128)
    out["aerial_perm"] = g.permutation
    out["aerial_aabb"] = np.stack([gr.aabb for gr in g.groups])
    waypoints = [(0, 0, 0), (60, 0, 0), (60, 50, 0), (120, 50, 0)]
    st = ss.generate_street_scene(seed=4, n_points=3000, trajectory_waypoints=waypoints, n_views=12,
                                  image_size=(80, 60), duration=5.0)
    out["street_positions"] = st.cloud.positions
    out["street_presence"] = st.cloud.timestamps
    out["street_cam_pos"] = np.stack([v.position for v in st.views])
    out["street_cam_rot"] = np.stack([v.rotation for v in st.views])
    out["street_cam_far"] = np.array([v.far for v in st.views])
    out["street_view_times"] = np.array([v.time for v in st.views])

    # ---- frusta (visibility.py:168-230) ------------------------------------
    for P in (1, 2, 3):
        fr = svis.patch_frusta(ds.views[4], P)
        out[f"frusta_P{P}"] = np.stack([f.planes for f in fr])

    # ---- access matrices (visibility.py:308-358) ---------------------------
    prng = np.random.default_rng(5)
    pg = prng.integers(0, 3, len(ds.cloud))[g.permutation]
    out["aerial_point_gpu"] = pg
    for P in (1, 2, 3):
        out[f"access_exact_P{P}"] = ss.build_access_matrix(g, pg, ds.views, P=P, granularity="exact")
        out[f"access_group_P{P}"] = ss.build_access_matrix(g, pg, ds.views, P=P, granularity="group_approx")
    # per-view visibility of the sorted cloud (full frustum, candidate groups only)
    vis = np.zeros(len(ds.cloud), dtype=np.uint32)
    for vi, view in enumerate(ds.views):
        fr = ss.frustum_from_view(view)
        idx = svis._candidate_indices(g, fr)
        m = svis.cull_points(fr, g.sorted_cloud.positions[idx])
        vis[idx[m]] |= np.uint32(1 << vi)
    out["aerial_vis_mask"] = vis
    # temporal street scene
    gs = ss.zorder_group(st.cloud, G=64)
    spg = np.random.default_rng(6).integers(0, 2, len(st.cloud))[gs.permutation]
    out["street_perm"] = gs.permutation
    out["street_point_gpu"] = spg
    out["street_access_temporal_P2"] = ss.build_access_matrix(gs, spg, st.views, P=2, temporal=True)
    out["street_access_spatial_P1"] = ss.build_access_matrix(gs, spg, st.views, P=1)

    # ---- bipartite graph + partitions (partition.py:65-534) ----------------
    graph = spart.build_bipartite_graph(g, ds)
    out["graph_group_weights"] = graph.group_weights
    out["graph_edge_groups"] = graph.edge_groups
    out["graph_edge_views"] = graph.edge_views
    out["graph_edge_weights"] = graph.edge_weights
    for parts in (2, 3):
        labels, q = spart.partition_graph(graph, parts, eps=0.05, seed=7)
        out[f"partition_labels_{parts}"] = labels
        out[f"partition_quality_{parts}"] = np.array([q.edge_cut, q.balance] + q.part_weights)
    for (M, Gm) in ((2, 2), (4, 1), (1, 4)):
        a = spart.hierarchical_partition(graph, M, Gm, eps=0.05, seed=5)
        out[f"hier_{M}x{Gm}_group_machine"] = a.group_machine
        out[f"hier_{M}x{Gm}_group_gpu"] = a.group_gpu
        out[f"hier_{M}x{Gm}_image_machine"] = a.image_machine
    # a larger synthetic graph exercising coarsening
    grng = np.random.default_rng(8)
    ng, nv = 300, 120
    eg, ev, ew = [], [], []
    for gi in range(ng):
        for vj in grng.choice(nv, size=grng.integers(1, 9), replace=False):
            eg.append(gi)
            ev.append(int(vj))
            ew.append(int(grng.integers(1, 50)))
    big = spart.BipartiteGraph(grng.integers(50, 200, ng).astype(np.int64), np.array(eg), np.array(ev),
                               np.array(ew), nv)
    out["big_group_weights"] = big.group_weights
    out["big_edge_groups"] = big.edge_groups
    out["big_edge_views"] = big.edge_views
    out["big_edge_weights"] = big.edge_weights
    out["big_n_views"] = np.array([nv])
    for parts in (2, 4, 8):
        labels, q = spart.partition_graph(big, parts, eps=0.05, seed=3)
        out[f"big_labels_{parts}"] = labels
        out[f"big_quality_{parts}"] = np.array([q.edge_cut, q.balance] + q.part_weights)
    labels, _ = spart.partition_graph(big, 4, eps=0.05, seed=3, image_weight_factor=0.5)
    out["big_labels_4_iwf"] = labels

    # ---- placement (placement.py:123-361) ----------------------------------
    mrng = np.random.default_rng(12)
    cases = []
    for ci in range(12):
        N = [2, 4, 8][ci % 3]
        B = N * int(mrng.integers(1, 5))
        mat = mrng.integers(0, 1000, (B, N)) * (mrng.uniform(0, 1, (B, N)) < 0.7)
        cases.append(mat.astype(np.int64))
    inter = splace.CostCoefficients(p=4.0)
    intra = splace.CostCoefficients(alpha=0.0, beta=0.1, gamma=0.1, delta=1.0, p=4.0)
    for ci, mat in enumerate(cases):
        out[f"place_mat_{ci}"] = mat
        B, N = mat.shape
        out[f"place_lsa_{ci}"] = splace.lsa_assign(mat, B // N).assignment
        sol, info = splace.local_search(mat, splace.lsa_assign(mat, B // N), splace.CostCoefficients())
        out[f"place_ls_{ci}"] = sol.assignment
        out[f"place_ls_hist_{ci}"] = np.array(info["relaxed_history"])
        out[f"place_flat_{ci}"] = splace.hierarchical_place(mat, 1, N, inter, intra).assignment
        if N % 2 == 0:
            out[f"place_hier_{ci}"] = splace.hierarchical_place(mat, 2, N // 2, inter, intra).assignment
        out[f"place_inf_{ci}"] = splace.place(mat, splace.CostCoefficients(p=np.inf)).assignment
        ob = splace.objective(mat, splace.PlacementSolution(out[f"place_flat_{ci}"], N), inter)
        out[f"place_obj_{ci}"] = np.array([ob.total_local, ob.exact_value, ob.relaxed_value])
        if splace._count_assignments(B, N, B // N) <= 20000:
            out[f"place_brute_{ci}"] = splace.brute_force_optimal(mat, inter).assignment

    # ---- simulator (simulator.py:134-423) ----------------------------------
    topo = ssim.ClusterTopology(machines=2, gpus_per_machine=2, inter_bandwidth=25e9, intra_bandwidth=300e9)
    for ci in (1, 4, 7):
        mat = cases[ci]
        N = mat.shape[1]
        sol = splace.PlacementSolution(out[f"place_flat_{ci}"], N)
        for M in sorted({1, 2, N}):
            if N % M:
                continue
            t2 = ssim.ClusterTopology(machines=M, gpus_per_machine=N // M, inter_bandwidth=25e9,
                                      intra_bandwidth=300e9)
            tr = ssim.account_iteration(mat, sol, t2, 44)
            out[f"trace_{ci}_M{M}"] = np.stack([tr.send_intra, tr.send_inter, tr.recv_intra, tr.recv_inter,
                                                tr.comp])
            out[f"trace_{ci}_M{M}_est"] = np.array([tr.est_time, tr.total_points])
    kw = dict(epochs=1, batch_size=4, P=2, seed=9)
    loc = ssim.LocalityAwareStrategy(group_size=128, seed=5, inter_coeffs=inter, intra_coeffs=intra)
    rep_r = ssim.run_training_sim(ds, topo, ssim.RandomStrategy(seed=5), **kw)
    rep_l = ssim.run_training_sim(ds, topo, loc, **kw)
    out["sim_random_json"] = np.frombuffer(json.dumps(rep_r.to_json(), sort_keys=True).encode(), dtype=np.uint8)
    out["sim_locality_json"] = np.frombuffer(json.dumps(rep_l.to_json(), sort_keys=True).encode(), dtype=np.uint8)
    out["sim_reduction"] = np.array([ssim.comm_reduction(rep_r, rep_l)])
    rnd = ssim._random_point_gpus(len(ds.cloud), 4, np.random.default_rng(np.random.SeedSequence([5, 17])))
    out["random_point_gpus"] = rnd
    out["random_placement"] = ssim._random_placement(16, 4, np.random.default_rng(
        np.random.SeedSequence([5, 3, 2]))).assignment

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
