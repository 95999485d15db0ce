"""Native multilevel partitioner (csrc/host/partition.cpp) vs the Python
restatement of the reference algorithm (oracle/py_partition.py): identical
labels on random geometric bipartite graphs (several sizes, part counts,
seeds), plus the scale it exists for."""

import time

import numpy as np
import pytest

from oracle.py_partition import Multilevel
from paper_2512_20017_b200 import sharding as sh


def _geo_graph(ng, nv, seed, radius=0.15):
    rng = np.random.default_rng(seed)
    gxy, vxy = rng.uniform(0, 1, (ng, 2)), rng.uniform(0, 1, (nv, 2))
    d = np.linalg.norm(gxy[:, None] - vxy[None], axis=2)
    gi, vi = np.nonzero(d < radius)
    w = rng.integers(1, 2048, len(gi))
    sizes = np.full(ng, 2048)
    sizes[-1] = 1 + seed % 2047
    return sh.BipartiteGraph(sizes, gi, vi, w, nv)


@pytest.mark.parametrize("ng,nv,parts,seed", [(60, 12, 2, 0), (300, 40, 3, 1), (900, 64, 4, 2), (1500, 96, 8, 3),
                                              (700, 50, 5, 4)])
def test_native_run_matches_python_restatement(ng, nv, parts, seed):
    g = sh._as_weighted(_geo_graph(ng, nv, seed), 0.0)
    for r in range(2):
        mk = lambda: np.random.default_rng(np.random.SeedSequence([seed, r]))  # noqa: E731
        ref = Multilevel(parts, 0.05, mk()).run(g)
        got = sh.multilevel_run(g, parts, 0.05, mk())
        assert np.array_equal(ref, got)


def test_native_run_image_weights():
    g = sh._as_weighted(_geo_graph(400, 30, 9), 0.5)
    mk = lambda: np.random.default_rng(np.random.SeedSequence([9, 0]))  # noqa: E731
    assert np.array_equal(Multilevel(4, 0.05, mk()).run(g), sh.multilevel_run(g, 4, 0.05, mk()))


def test_native_partition_scales():
    """25k groups x 256 views (C4-sized graph): one run in seconds."""
    graph = _geo_graph(25_000, 256, 11, radius=0.08)
    t = time.perf_counter()
    lab, q = sh.partition_graph(graph, 8, eps=0.05, seed=5, runs=1)
    dt = time.perf_counter() - t
    assert q.balance <= 1.05 + 1e-9
    assert len(np.unique(lab[:25_000])) == 8
    assert dt < 120.0, dt
