"""Points-to-rank partitioner (offline point placement).

Public contract of /root/reference/pkg/src/splatsched/partition.py:
``BipartiteGraph``, ``build_bipartite_graph``, ``partition_graph``,
``evaluate_partition``, ``hierarchical_partition``, ``PartitionAssignment``,
``image_ownership``.  The (group, view) visible-point counts that weight the
graph are computed by the sm_100a culling kernel in edge mode (one launch
per chunk of views instead of the reference's Python loop over views x
groups, partition.py:74-89).  The multilevel k-way partitioner is a host
algorithm that consumes numpy PCG64 draws; it reproduces the reference's
labels exactly (same draw sequence, same tie-breaking); it runs in the
native host library (csrc/host/partition.cpp, include/splat_host.h):
  coarsening   heavy-edge matching, vertices in index order, ties among
               equally heavy free neighbours broken by rng.integers
               (partition.py:133-186)
  initial      greedy growth of parts 0..k-2 from random seeds, leftovers to
               part k-1 (partition.py:189-223)
  refinement   forced rebalance, then greedy single-vertex moves: strictly
               positive cut gain first (lowest (v, t)), else a zero-gain move
               that strictly lowers the sum of squared part weights
               (partition.py:248-327)
  runs         best of `runs` seeds by (cut, balance, run) (partition.py:398-434)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .status import ConsistencyError, InfeasiblePartitionError, ParameterError

DEFAULT_EPSILON = 0.05
DEFAULT_RUNS = 4
COARSEN_FACTOR = 30


@dataclass
class BipartiteGraph:
    """Point-group vertices (weight = size) x view vertices; edge weight = the
    number of the group's points visible in the view (>= 1)."""

    group_weights: np.ndarray
    edge_groups: np.ndarray
    edge_views: np.ndarray
    edge_weights: np.ndarray
    n_views: int

    @property
    def n_groups(self) -> int:
        return len(self.group_weights)

    @property
    def view_weights(self) -> np.ndarray:
        w = np.zeros(self.n_views, dtype=np.int64)
        np.add.at(w, self.edge_views, self.edge_weights)
        return w

    @property
    def n_vertices(self) -> int:
        return self.n_groups + self.n_views


def group_view_counts(grouped, views, temporal: bool = False) -> np.ndarray:
    """int32 [n_groups, n_views]: visible points of every group in every
    full-view frustum (K0 edge mode, AABB early-out per group)."""
    from .culling import _dev, batch_planes

    dev = _dev()
    pos, gbeg, aabb, pres = grouped.device_arrays(dev)
    ng = grouped.n_groups
    out = torch.zeros((ng, len(views)), dtype=torch.int32, device=dev)
    chunk = 256
    for s in range(0, len(views), chunk):
        vs = views[s:s + chunk]
        planes = torch.as_tensor(batch_planes(vs, 1), device=dev)
        vt = torch.as_tensor(np.array([v.time for v in vs], dtype=np.float32), device=dev) if temporal else None
        part = torch.empty((ng, len(vs)), dtype=torch.int32, device=dev)
        nat.call("bs_cull_count", nat.CullDesc(nat.CULL_EDGES, len(vs), 1, 1, 1 if temporal else 0, 3), nat.ptr(pos),
                 len(pos), nat.ptr(pres) if temporal else None, nat.ptr(gbeg), nat.ptr(aabb), ng, nat.ptr(planes),
                 nat.ptr(vt), None, nat.ptr(part), None, None, nat.stream_handle())
        out[:, s:s + len(vs)] = part
    return out.cpu().numpy()


def build_bipartite_graph(grouped, dataset) -> BipartiteGraph:
    """Exact (group, view) visible counts for the whole dataset; edges in
    view-major order like the reference loop (partition.py:74-89)."""
    if len(grouped.sorted_cloud) != len(dataset.cloud):
        raise ConsistencyError("grouped cloud does not match dataset cloud")
    counts = group_view_counts(grouped, dataset.views, temporal=dataset.profile.temporal)
    ev, eg = np.nonzero(counts.T)
    return BipartiteGraph(
        group_weights=np.array([g.size for g in grouped.groups], dtype=np.int64),
        edge_groups=eg.astype(np.int64),
        edge_views=np.array([dataset.views[v].id for v in ev], dtype=np.int64),
        edge_weights=counts.T[ev, eg].astype(np.int64),
        n_views=len(dataset.views),
    )


# ---------------------------------------------------------------------------
# weighted graph + multilevel k-way partitioner


class WeightedGraph:
    """Undirected graph: CSR adjacency (neighbours ascending) + edge list."""

    def __init__(self, n, balance, eu, ev, ew):
        self.n = n
        self.bal = np.asarray(balance, dtype=np.float64)
        self.eu = np.asarray(eu, dtype=np.int64)
        self.ev = np.asarray(ev, dtype=np.int64)
        self.ew = np.asarray(ew, dtype=np.float64)
        src = np.concatenate([self.eu, self.ev])
        dst = np.concatenate([self.ev, self.eu])
        wt = np.concatenate([self.ew, self.ew])
        order = np.lexsort((dst, src))
        self.adj = dst[order]
        self.adj_w = wt[order]
        self.ptr = np.concatenate([[0], np.cumsum(np.bincount(src, minlength=n))]).astype(np.int64)

    def nbrs(self, v):
        a, b = self.ptr[v], self.ptr[v + 1]
        return self.adj[a:b], self.adj_w[a:b]

    def cut(self, labels) -> float:
        return float(self.ew[labels[self.eu] != labels[self.ev]].sum())

    def part_weights(self, labels, parts):
        w = np.zeros(parts)
        np.add.at(w, labels, self.bal)
        return w


def _pcg_state(rng: np.random.Generator) -> np.ndarray:
    """numpy PCG64 state as {state_hi, state_lo, inc_hi, inc_lo, has_uint32,
    uinteger} (include/splat_host.h)."""
    st = rng.bit_generator.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]), int(st["uinteger"])],
                    dtype=np.uint64)


def multilevel_run(g: WeightedGraph, parts: int, eps: float, rng: np.random.Generator) -> np.ndarray:
    """One run of the multilevel k-way scheme (partition.py:104-434) in the
    native host library (csrc/host/partition.cpp): same decisions and the
    same PCG64 draws as the reference, so identical labels."""
    n = int(g.n)
    bal = np.ascontiguousarray(g.bal, dtype=np.float64)
    eu = np.ascontiguousarray(g.eu, dtype=np.int64)
    ev = np.ascontiguousarray(g.ev, dtype=np.int64)
    ew = np.ascontiguousarray(g.ew, dtype=np.float64)
    state = _pcg_state(rng)
    lab = np.empty(n, dtype=np.int64)
    nat.host_call("bs_partition_multilevel", n, bal.ctypes.data, len(eu), eu.ctypes.data, ev.ctypes.data,
                  ew.ctypes.data, int(parts), float(eps), state.ctypes.data, lab.ctypes.data)
    return lab


@dataclass
class PartitionQuality:
    edge_cut: float
    balance: float
    part_weights: list

    def to_json(self) -> dict:
        return {"edge_cut": self.edge_cut, "balance": self.balance, "part_weights": self.part_weights}


def _as_weighted(graph: BipartiteGraph, image_weight_factor: float) -> WeightedGraph:
    bal = np.concatenate([graph.group_weights.astype(np.float64),
                          image_weight_factor * graph.view_weights.astype(np.float64)])
    return WeightedGraph(graph.n_vertices, bal, graph.edge_groups, graph.edge_views + graph.n_groups,
                         graph.edge_weights)


def evaluate_partition(graph: BipartiteGraph, labels, parts, image_weight_factor=0.0) -> PartitionQuality:
    g = _as_weighted(graph, image_weight_factor)
    labels = np.asarray(labels, dtype=np.int64)
    pw = g.part_weights(labels, parts)
    mean = g.bal.sum() / parts
    return PartitionQuality(g.cut(labels), float(pw.max() / mean) if mean > 0 else 1.0, [float(x) for x in pw])


def partition_graph(graph: BipartiteGraph, parts: int, eps: float = DEFAULT_EPSILON, seed: int = 0,
                    runs: int = DEFAULT_RUNS, image_weight_factor: float = 0.0):
    """Labels over n_groups + n_views vertices and their PartitionQuality."""
    if parts < 1:
        raise ParameterError("parts must be >= 1")
    if graph.n_vertices == 0:
        raise ParameterError("graph is empty")
    g = _as_weighted(graph, image_weight_factor)
    if parts == 1:
        lab = np.zeros(g.n, dtype=np.int64)
        return lab, evaluate_partition(graph, lab, 1, image_weight_factor)
    cap = (1.0 + eps) * g.bal.sum() / parts
    heavy = int(np.argmax(g.bal))
    if g.bal[heavy] > cap:
        raise InfeasiblePartitionError(f"vertex {heavy} (weight {g.bal[heavy]:g}) exceeds the balance cap "
                                       f"{cap:g}; no {parts}-way partition satisfies eps={eps}")
    best = None
    for r in range(runs):
        lab = multilevel_run(g, parts, eps, np.random.default_rng(np.random.SeedSequence([int(seed), r])))
        q = evaluate_partition(graph, lab, parts, image_weight_factor)
        key = (q.edge_cut, q.balance, r)
        if best is None or key < best[0]:
            best = (key, lab, q)
    return best[1], best[2]


@dataclass
class PartitionAssignment:
    """group -> (machine, gpu), plus the image vertices' machine labels."""

    group_machine: np.ndarray
    group_gpu: np.ndarray
    machines: int
    gpus_per_machine: int
    group_weights: np.ndarray
    image_machine: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))

    @property
    def n_groups(self) -> int:
        return len(self.group_machine)

    @property
    def n_gpus(self) -> int:
        return self.machines * self.gpus_per_machine

    def flat_gpu(self, group_id: int) -> int:
        return int(self.group_machine[group_id] * self.gpus_per_machine + self.group_gpu[group_id])

    def flat_gpus(self) -> np.ndarray:
        return self.group_machine * self.gpus_per_machine + self.group_gpu

    def per_gpu_weights(self) -> np.ndarray:
        w = np.zeros(self.n_gpus, dtype=np.int64)
        np.add.at(w, self.flat_gpus(), self.group_weights)
        return w


def hierarchical_partition(graph: BipartiteGraph, machines: int, gpus_per_machine: int,
                           eps: float = DEFAULT_EPSILON, seed: int = 0) -> PartitionAssignment:
    """Machine-level partition of the whole graph, then a GPU-level partition
    of each machine's induced subgraph (seed + machine * 1000003)."""
    if machines < 1 or gpus_per_machine < 1:
        raise ParameterError("machines and gpus_per_machine must be >= 1")
    ng = graph.n_groups
    top, _ = partition_graph(graph, machines, eps, seed)
    group_machine = top[:ng].copy()
    image_machine = top[ng:].copy()
    # each image joins the machine holding most of its visible points
    inc = np.zeros((graph.n_views, machines))
    np.add.at(inc, (graph.edge_views, group_machine[graph.edge_groups]), graph.edge_weights)
    home = np.where(inc.sum(axis=1) > 0, np.argmax(inc, axis=1), image_machine)
    group_gpu = np.zeros(ng, dtype=np.int64)
    if gpus_per_machine > 1:
        for m in range(machines):
            gs = np.flatnonzero(group_machine == m)
            if len(gs) == 0:
                continue
            vs = np.flatnonzero(home == m)
            sel = np.isin(graph.edge_groups, gs) & np.isin(graph.edge_views, vs)
            sub = BipartiteGraph(graph.group_weights[gs], np.searchsorted(gs, graph.edge_groups[sel]),
                                 np.searchsorted(vs, graph.edge_views[sel]), graph.edge_weights[sel], len(vs))
            lab, _ = partition_graph(sub, gpus_per_machine, eps, int(seed) + m * 1000003)
            group_gpu[gs] = lab[:len(gs)]
    return PartitionAssignment(group_machine, group_gpu, machines, gpus_per_machine, graph.group_weights.copy(),
                               image_machine)


def image_ownership(assignment: PartitionAssignment, graph: BipartiteGraph):
    if len(assignment.image_machine) != graph.n_views:
        raise ConsistencyError("assignment image labels do not match graph views")
    return {v: int(assignment.image_machine[v]) for v in range(graph.n_views)}
