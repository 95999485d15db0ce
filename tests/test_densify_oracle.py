"""CPU oracle of the densification step (oracle/splat_oracle.c so_densify_*,
the restatement of csrc/densify.cu; PAPER.md:273 periodic densification, 3DGS
clone / split / prune): structural properties of the new shard.  The GPU
kernels are compared with it bit for bit in tests/test_gpu_densify.py."""

import numpy as np

from oracle import py_oracle

from _densify import CFG, densify_inputs


def test_densify_oracle_actions_and_layout():
    ds, params, gb, aabb, gt, stats, m, v = densify_inputs()
    act, gout, nb, pn, mn, vn, src, aabb_n = py_oracle.densify(params, m, v, stats, gb, CFG["grad_threshold"],
                                                               CFG["split_scale"], CFG["min_opacity"],
                                                               CFG["max_scale"], CFG["seed"])
    S = params.shape[1]
    counts = np.bincount(act, minlength=4)
    assert all(counts > 100), counts  # every action occurs
    assert nb[-1] == counts[1] + 2 * counts[2] + 2 * counts[3] == pn.shape[1]
    # rules: prune by opacity, densify by the mean statistic, split vs clone by the largest scale
    o = 1.0 / (1.0 + np.exp(-params[0, :, 3].astype(np.float64)))
    smax = np.exp(params[1, :, :3].astype(np.float64)).max(axis=1)
    avg = np.where(stats[:, 1] > 0, stats[:, 0] / np.maximum(stats[:, 1], 1), 0.0)
    clear = (np.abs(o - CFG["min_opacity"]) > 1e-4) & (np.abs(avg - CFG["grad_threshold"]) > 1e-7) & \
        (np.abs(smax - CFG["split_scale"]) > 1e-4)
    want = np.where(o < CFG["min_opacity"], 0, np.where(avg >= CFG["grad_threshold"],
                                                        np.where(smax > CFG["split_scale"], 3, 2), 1))
    assert np.array_equal(act[clear], want[clear])
    # outputs stay in their group, in point order
    for g in range(len(gb) - 1):
        s = src[nb[g]:nb[g + 1]]
        assert np.all((s >= gb[g]) & (s < gb[g + 1])) and np.all(np.diff(s) >= 0)
    # keep / clone: exact copies; the clone carries zero moments; split children: zero moments,
    # log scale - ln 1.6, rotation/opacity/SH copied, means displaced ~ N(0, s^2) along the axes
    first = np.ones(len(src), bool)
    first[1:] = src[1:] != src[:-1]
    a_of = act[src]
    kc = (a_of == 1) | (a_of == 2)
    assert np.array_equal(pn[:, kc], params[:, src[kc]])
    orig = kc & first
    assert np.array_equal(mn[:, orig], m[:, src[orig]]) and np.array_equal(vn[:, orig], v[:, src[orig]])
    assert not mn[:, kc & ~first].any() and not vn[:, kc & ~first].any()
    sp = a_of == 3
    assert not mn[:, sp].any() and not vn[:, sp].any()
    assert np.array_equal(pn[1, sp, :3], (params[1, src[sp], :3] - np.float32(np.log(1.6))).astype(np.float32))
    assert np.array_equal(pn[2:, sp], params[2:, src[sp]]) and np.array_equal(pn[0, sp, 3], params[0, src[sp], 3])
    # displacement in the point's local frame, standardised by its scales: ~ N(0, 1)
    q = params[2, src[sp]].astype(np.float64)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    R = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                  2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                  2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], axis=1).reshape(-1, 3, 3)
    d = pn[0, sp, :3].astype(np.float64) - params[0, src[sp], :3].astype(np.float64)
    eps = np.einsum("nji,nj->ni", R, d) / np.exp(params[1, src[sp], :3].astype(np.float64))
    assert abs(eps.mean()) < 0.05 and abs(eps.std() - 1.0) < 0.05 and np.abs(eps).max() <= 6.0
    # the two children of a split differ
    assert not np.array_equal(pn[0, sp][0::2], pn[0, sp][1::2])
    # group AABBs bound the new means exactly
    for g in range(len(gb) - 1):
        p = pn[0, nb[g]:nb[g + 1], :3]
        if len(p):
            assert np.array_equal(aabb_n[g], np.concatenate([p.min(axis=0), p.max(axis=0)]))


def test_densify_oracle_deterministic_and_keyed_by_global_id():
    ds, params, gb, aabb, gt, stats, m, v = densify_inputs()
    args = (CFG["grad_threshold"], CFG["split_scale"], CFG["min_opacity"], CFG["max_scale"])
    a = py_oracle.densify(params, m, v, stats, gb, *args, seed=3)
    b = py_oracle.densify(params, m, v, stats, gb, *args, seed=3)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    c = py_oracle.densify(params, m, v, stats, gb, *args, seed=4)
    assert np.array_equal(a[0], c[0]) and not np.array_equal(a[3], c[3])  # same actions, other samples
    gid = np.arange(params.shape[1], dtype=np.int32) * 3 + 5
    d = py_oracle.densify(params, m, v, stats, gb, *args, seed=3, gid=gid)
    assert not np.array_equal(a[3], d[3])
    # no statistics: nothing densifies, only pruning
    e = py_oracle.densify(params, m, v, None, gb, *args)
    assert set(np.unique(e[0])) <= {0, 1}
