"""Shared inputs of the densification tests: a C1 shard with statistics that
exercise every action (prune, keep, clone, split)."""

import numpy as np

from _scene import c1_setup

CFG = dict(grad_threshold=2e-4, split_scale=1.0, min_opacity=0.05, max_scale=0.0, seed=7)


def densify_inputs():
    ds, params, gb, aabb, gt = c1_setup()
    params = params.copy()
    S = params.shape[1]
    rng = np.random.default_rng(11)
    # opacities low enough to prune ~10 %, scales on both sides of split_scale
    low = rng.random(S) < 0.1
    params[0, low, 3] = -4.0                                 # sigmoid ~ 0.018 < 0.05
    big = rng.random(S) < 0.3
    params[1, big, :3] = np.log(rng.uniform(1.2, 2.0, (int(big.sum()), 3))).astype(np.float32)
    stats = np.zeros((S, 2), np.float32)
    seen = rng.random(S) < 0.8
    stats[seen, 1] = rng.integers(1, 5, int(seen.sum()))
    stats[seen, 0] = stats[seen, 1] * rng.uniform(0.0, 4e-4, int(seen.sum())).astype(np.float32)
    m = rng.normal(0, 1e-3, params.shape).astype(np.float32)
    v = rng.uniform(0, 1e-6, params.shape).astype(np.float32)
    return ds, params, gb, aabb, gt, stats, m, v
