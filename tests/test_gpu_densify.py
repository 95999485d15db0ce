"""Densification on the GPU (csrc/densify.cu; PAPER.md:273 periodic
densification, standard 3DGS clone / split / prune) against the CPU oracle
(oracle/splat_oracle.c so_densify_*):
  * actions, group table, new parameters / Adam moments, source indices and
    group AABBs: bit-exact (the split samples are integer hashes and every
    float op is round-to-nearest on both sides);
  * the statistic the fused projection backward accumulates: the NDC-space
    |dL/d mean2d| of every (point, view) recomputed from the step's own G_SP
    and SP rows, within 1e-5;
  * a training step on the densified shard matches the oracle pipeline run on
    that shard (SP rows and per-tile lists bit-exact, image <= 1e-4, G_SP
    <= 1e-4 x per-component max)."""

import numpy as np
import pytest
import torch

from paper_2512_20017_b200 import _native as nat
from paper_2512_20017_b200.trainer import DensifyConfig, SplatTrainer, camera_bytes

from _densify import CFG, densify_inputs
from _scene import oracle_view_pipeline

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def inputs(cuda):
    return densify_inputs()


def _gpu_densify(params, m, v, stats, gb, gid=None, seed=CFG["seed"]):
    dev = torch.device("cuda")
    S, ng = params.shape[1], len(gb) - 1
    P, M, V = (torch.as_tensor(a, device=dev) for a in (params, m, v))
    st = torch.as_tensor(stats, device=dev)
    g = torch.as_tensor(np.asarray(gb, np.int32), device=dev)
    G = None if gid is None else torch.as_tensor(gid, device=dev)
    desc = nat.DensifyDesc(nat.MODEL_3DGS, CFG["grad_threshold"], CFG["split_scale"], CFG["min_opacity"],
                           CFG["max_scale"], seed)
    act = torch.empty(S, dtype=torch.int32, device=dev)
    gout = torch.empty(ng, dtype=torch.int32, device=dev)
    nat.call("bs_densify_mark", desc, nat.ptr(P), S, nat.ptr(st), nat.ptr(g), ng, nat.ptr(act), nat.ptr(gout), None)
    nb = torch.zeros(ng + 1, dtype=torch.int32, device=dev)
    nb[1:] = torch.cumsum(gout, 0, dtype=torch.int32)
    Sn = int(nb[-1])
    pn, mn, vn = (torch.empty(15, Sn, 4, device=dev) for _ in range(3))
    src = torch.empty(Sn, dtype=torch.int32, device=dev)
    nat.call("bs_densify_apply", desc, nat.ptr(P), nat.ptr(M), nat.ptr(V), S, nat.ptr(act), nat.ptr(g), nat.ptr(nb),
             ng, nat.ptr(G), nat.ptr(pn), nat.ptr(mn), nat.ptr(vn), Sn, nat.ptr(src), None)
    aabb = torch.empty(ng, 6, device=dev)
    nat.call("bs_group_aabb_ranges", nat.ptr(pn), Sn, nat.ptr(nb), ng, nat.ptr(aabb), None)
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in (act, gout, nb, pn, mn, vn, src, aabb)]


@pytest.mark.parametrize("with_gid", [False, True])
def test_densify_kernels_bitexact_vs_oracle(inputs, with_gid):
    from oracle import py_oracle

    ds, params, gb, aabb, gt, stats, m, v = inputs
    gid = (np.arange(params.shape[1], dtype=np.int32) * 2 + 1) if with_gid else None
    mine = _gpu_densify(params, m, v, stats, gb, gid)
    ref = py_oracle.densify(params, m, v, stats, gb, CFG["grad_threshold"], CFG["split_scale"], CFG["min_opacity"],
                            CFG["max_scale"], CFG["seed"], gid=gid)
    names = ("action", "group_out", "group_begin", "params", "exp_avg", "exp_avg_sq", "src_index", "aabb")
    for name, a, b in zip(names, mine, ref):
        assert a.shape == b.shape, name
        assert np.array_equal(a.view(np.uint32) if a.dtype == np.float32 else a,
                              b.view(np.uint32) if b.dtype == np.float32 else b), name
    assert all(np.bincount(ref[0], minlength=4) > 100)


def test_densify_statistic_accumulation(c1_trainer):
    tr = c1_trainer
    tr.track_densify_stats(True)
    tr.record_row_gid = True
    batch = [0, 2, 5, 7]
    tr.step(batch)
    stats = tr.densify_stats.cpu().numpy()
    n = tr.last["n_rows"]
    sp = tr.last["sp"][: n * 12].cpu().numpy().reshape(-1, 12).astype(np.float64)
    gsp = tr.last["gsp"][: n * 12].cpu().numpy().reshape(-1, 12).astype(np.float64)
    rows_gid = tr.last["row_gid"][:n].cpu().numpy() if "row_gid" in tr.last else None
    assert rows_gid is not None
    A, B, C = sp[:, 3], sp[:, 4], sp[:, 5]
    gu = -(A * gsp[:, 0] + B * gsp[:, 1])
    gv = -(B * gsp[:, 0] + C * gsp[:, 1])
    norm = np.hypot(gu * tr.W / 2, gv * tr.H / 2)
    valid = (sp[:, 10] > 0) | (sp[:, 11] > 0)
    exp = np.zeros((tr.S, 2))
    np.add.at(exp[:, 0], rows_gid[valid], norm[valid])
    np.add.at(exp[:, 1], rows_gid[valid], 1.0)
    assert np.array_equal(stats[:, 1], exp[:, 1])
    scale = np.abs(exp[:, 0]).max()
    assert scale > 0 and np.abs(stats[:, 0] - exp[:, 0]).max() <= 1e-5 * scale


@pytest.fixture
def c1_trainer(inputs):
    ds, params, gb, aabb, gt, stats, m, v = inputs
    from _scene import c1_setup

    ds, params, gb, aabb, gt = c1_setup()
    return SplatTrainer(params, gb, aabb, ds.views, gt=gt, sh_degree=3)


def test_densify_then_train_matches_oracle(c1_trainer):
    from oracle import py_oracle

    tr = c1_trainer
    ds_views = tr.views
    tr.track_densify_stats(True)
    for batch in ([0, 2, 5, 7], [1, 3, 4, 6]):
        tr.step(batch)
    p0, m0, v0 = (t.cpu().numpy().copy() for t in (tr.params, tr.exp_avg, tr.exp_avg_sq))
    st = tr.densify_stats.cpu().numpy().copy()
    gb0 = tr.group_begin.cpu().numpy().copy()
    thr = float(np.quantile(st[:, 0] / np.maximum(st[:, 1], 1), 0.8))  # densify the top ~20 %
    cfg = DensifyConfig(grad_threshold=thr, split_scale=1.0, min_opacity=0.05, seed=1)
    rep = tr.densify(cfg)
    ref = py_oracle.densify(p0, m0, v0, st, gb0, thr, 1.0, 0.05, 0.0, 1)
    assert rep["n_after"] == tr.S == ref[3].shape[1] and rep["n_after"] > rep["n_before"]
    assert rep["cloned"] > 0 and rep["split"] > 0
    assert np.array_equal(tr.params.cpu().numpy().view(np.uint32), ref[3].view(np.uint32))
    assert np.array_equal(tr.exp_avg.cpu().numpy(), ref[4]) and np.array_equal(tr.exp_avg_sq.cpu().numpy(), ref[5])
    assert np.array_equal(tr.group_begin.cpu().numpy(), ref[2])
    assert np.array_equal(tr.aabb.cpu().numpy().view(np.uint32), ref[7].view(np.uint32))
    assert not tr.densify_stats.any()
    # a step on the densified shard == the oracle pipeline on that shard
    params = tr.params.cpu().numpy().copy()
    gb, aabb = ref[2], ref[7]
    gt = tr.gt.cpu().numpy()
    batch = [1, 6]
    losses = tr.step(batch).cpu().numpy()
    n = tr.last["n_rows"]
    H, W = tr.H, tr.W
    rows = tr.last["rows_per_view"]
    row0 = np.concatenate([[0], np.cumsum(rows)])
    sp = tr.last["sp"][: n * 12].cpu().numpy().reshape(-1, 12)
    img = tr.last["image"][: len(batch) * H * W * 3].cpu().numpy().reshape(len(batch), H, W, 3)
    g = tr.last["gsp"][: n * 12].cpu().numpy().reshape(-1, 12)[:, :9]
    T = tr.tiles
    irows = tr.last["irows"][: tr.last["n_inst"]].cpu().numpy().astype(np.int64)
    for s, vid in enumerate(batch):
        r = oracle_view_pipeline(params, gb, aabb, ds_views[vid], camera_bytes([ds_views[vid]]), gt[vid])
        assert np.array_equal(sp[row0[s]:row0[s + 1]].view(np.uint32), r["sp"].view(np.uint32))
        rr = tr.last["ranges"][s * T * 2:(s + 1) * T * 2].cpu().numpy().reshape(T, 2)
        lens = rr[:, 1] - rr[:, 0]
        assert np.array_equal(lens, r["ranges"][:, 1] - r["ranges"][:, 0])
        nz = np.flatnonzero(lens)
        mine = np.concatenate([irows[rr[t, 0]:rr[t, 1]] for t in nz]) - row0[s]
        theirs = np.concatenate([r["lists"][r["ranges"][t, 0]:r["ranges"][t, 1]] for t in nz]).astype(np.int64)
        assert np.array_equal(mine, theirs)
        assert np.abs(img[s] - r["img"]).max() <= 1e-4
        assert abs(losses[s] - r["loss"]) <= 1e-5
        scale = np.abs(r["gsp"]).max(axis=0) + 1e-30
        assert ((np.abs(g[row0[s]:row0[s + 1]] - r["gsp"]) / scale).max(axis=0) <= 1e-4).all()
    # and training goes on
    for batch in ([0, 3], [2, 5, 7]):
        assert np.isfinite(tr.step(batch).cpu().numpy()).all()


def test_densified_checkpoint_resumes(c1_trainer, tmp_path):
    """state_dict after densification carries the new shard layout; a trainer
    built on the original shard resumes from it and steps exactly like the
    densified one (same kernels, same inputs)."""
    from _scene import c1_setup

    tr = c1_trainer
    tr.track_densify_stats(True)
    tr.step([0, 2, 5, 7])
    st = tr.densify_stats.cpu().numpy()
    thr = float(np.quantile(st[:, 0] / np.maximum(st[:, 1], 1), 0.7))
    tr.densify(DensifyConfig(grad_threshold=thr, split_scale=1.0, min_opacity=0.05, seed=2))
    tr.step([1, 3])
    torch.save(tr.state_dict(), tmp_path / "ckpt.pt")
    ds, params, gb, aabb, gt = c1_setup()
    b = SplatTrainer(params, gb, aabb, ds.views, gt=gt, sh_degree=3)
    b.load_state_dict(torch.load(tmp_path / "ckpt.pt"))
    assert b.S == tr.S != params.shape[1] and b.step_count == tr.step_count
    assert b.densify_stats is not None and torch.equal(b.densify_stats, tr.densify_stats)
    la = tr.step([4, 6]).cpu().numpy()
    lb = b.step([4, 6]).cpu().numpy()
    assert np.array_equal(la, lb)
    n = tr.last["n_rows"]
    assert torch.equal(tr.last["sp"][: n * 12], b.last["sp"][: n * 12])
