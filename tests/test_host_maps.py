"""CPU parity of the host-side maps against the reference's golden vectors:
points-to-rank partition labels, image-to-rank assignments, transfer
accounting and the random baseline (bit-exact)."""

import numpy as np
import pytest

from paper_2512_20017_b200 import accounting as acc
from paper_2512_20017_b200 import assign as asg
from paper_2512_20017_b200 import sharding as sh

INTER = asg.CostCoefficients(p=4.0)
INTRA = asg.CostCoefficients(alpha=0.0, beta=0.1, gamma=0.1, delta=1.0, p=4.0)


def _graph(golden, prefix="graph"):
    if prefix == "graph":
        return sh.BipartiteGraph(golden["graph_group_weights"], golden["graph_edge_groups"],
                                 golden["graph_edge_views"], golden["graph_edge_weights"], 10)
    return sh.BipartiteGraph(golden["big_group_weights"], golden["big_edge_groups"], golden["big_edge_views"],
                             golden["big_edge_weights"], int(golden["big_n_views"][0]))


@pytest.mark.parametrize("parts", [2, 3])
def test_partition_graph_matches_reference(golden, parts):
    labels, q = sh.partition_graph(_graph(golden), parts, eps=0.05, seed=7)
    assert np.array_equal(labels, golden[f"partition_labels_{parts}"])
    assert np.array_equal(np.array([q.edge_cut, q.balance] + q.part_weights), golden[f"partition_quality_{parts}"])


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_partition_graph_multilevel_matches_reference(golden, parts):
    labels, q = sh.partition_graph(_graph(golden, "big"), parts, eps=0.05, seed=3)
    assert np.array_equal(labels, golden[f"big_labels_{parts}"])
    assert np.array_equal(np.array([q.edge_cut, q.balance] + q.part_weights), golden[f"big_quality_{parts}"])


def test_partition_image_weight_factor(golden):
    labels, _ = sh.partition_graph(_graph(golden, "big"), 4, eps=0.05, seed=3, image_weight_factor=0.5)
    assert np.array_equal(labels, golden["big_labels_4_iwf"])


@pytest.mark.parametrize("M,Gm", [(2, 2), (4, 1), (1, 4)])
def test_hierarchical_partition_matches_reference(golden, M, Gm):
    a = sh.hierarchical_partition(_graph(golden), M, Gm, eps=0.05, seed=5)
    assert np.array_equal(a.group_machine, golden[f"hier_{M}x{Gm}_group_machine"])
    assert np.array_equal(a.group_gpu, golden[f"hier_{M}x{Gm}_group_gpu"])
    assert np.array_equal(a.image_machine, golden[f"hier_{M}x{Gm}_image_machine"])


def test_partition_errors(golden):
    g = _graph(golden)
    with pytest.raises(sh.ParameterError):
        sh.partition_graph(g, 0)
    with pytest.raises(sh.InfeasiblePartitionError):
        sh.partition_graph(sh.BipartiteGraph(np.array([100, 1]), np.array([0]), np.array([0]), np.array([1]), 1), 2)


@pytest.mark.parametrize("ci", range(12))
def test_placement_matches_reference(golden, ci):
    mat = golden[f"place_mat_{ci}"]
    B, N = mat.shape
    assert np.array_equal(asg.lsa_assign(mat, B // N).assignment, golden[f"place_lsa_{ci}"])
    for native in (False, True):  # numpy restatement and the C++/OpenMP search (csrc/host/placement.cpp)
        sol, info = asg.local_search(mat, asg.lsa_assign(mat, B // N), asg.CostCoefficients(), native=native)
        assert np.array_equal(sol.assignment, golden[f"place_ls_{ci}"])
        assert np.array_equal(np.array(info["relaxed_history"]), golden[f"place_ls_hist_{ci}"])
    flat = asg.hierarchical_place(mat, 1, N, INTER, INTRA)
    assert np.array_equal(flat.assignment, golden[f"place_flat_{ci}"])
    if N % 2 == 0:
        assert np.array_equal(asg.hierarchical_place(mat, 2, N // 2, INTER, INTRA).assignment,
                              golden[f"place_hier_{ci}"])
    assert np.array_equal(asg.place(mat, asg.CostCoefficients(p=np.inf)).assignment, golden[f"place_inf_{ci}"])
    ob = asg.objective(mat, asg.PlacementSolution(golden[f"place_flat_{ci}"], N), INTER)
    assert np.array_equal(np.array([ob.total_local, ob.exact_value, ob.relaxed_value]), golden[f"place_obj_{ci}"])
    if f"place_brute_{ci}" in golden:
        assert np.array_equal(asg.brute_force_optimal(mat, INTER).assignment, golden[f"place_brute_{ci}"])


def test_single_box_topologies_give_identical_assignment(golden):
    """(1, N) and (N, 1) produce the same W."""
    for ci in range(12):
        mat = golden[f"place_mat_{ci}"]
        N = mat.shape[1]
        a = asg.hierarchical_place(mat, 1, N, INTER, INTRA).assignment
        b = asg.hierarchical_place(mat, N, 1, INTER, INTRA).assignment
        assert np.array_equal(a, b)


@pytest.mark.parametrize("ci", [1, 4, 7])
def test_account_iteration_matches_reference(golden, ci):
    mat = golden[f"place_mat_{ci}"]
    N = mat.shape[1]
    sol = asg.PlacementSolution(golden[f"place_flat_{ci}"], N)
    for M in sorted({1, 2, N}):
        if N % M:
            continue
        topo = acc.ClusterTopology(M, N // M, 25e9, 300e9)
        tr = acc.account_iteration(mat, sol, topo, 44)
        got = np.stack([tr.send_intra, tr.send_inter, tr.recv_intra, tr.recv_inter, tr.comp])
        assert np.array_equal(got, golden[f"trace_{ci}_M{M}"])
        assert np.array_equal(np.array([tr.est_time, tr.total_points]), golden[f"trace_{ci}_M{M}_est"])
        # conservation laws (test_acceptance.py:275-300)
        assert tr.send_intra.sum() == tr.recv_intra.sum() and tr.send_inter.sum() == tr.recv_inter.sum()
        assert tr.comp.sum() == mat.sum()


def test_random_baseline_maps(golden):
    rng = np.random.default_rng(np.random.SeedSequence([5, 17]))
    assert np.array_equal(acc.random_point_gpus(6000, 4, rng), golden["random_point_gpus"])
    rng = np.random.default_rng(np.random.SeedSequence([5, 3, 2]))
    assert np.array_equal(acc.random_placement(16, 4, rng).assignment, golden["random_placement"])


def test_comm_reduction_schedule_check():
    topo = acc.ClusterTopology(2, 1, 1e9, 1e9)
    r1 = acc.EpochReport("a", 0, 1, 1, 1, topo, [], [[0]])
    r2 = acc.EpochReport("b", 0, 1, 1, 1, topo, [], [[1]])
    with pytest.raises(acc.ComparisonError):
        acc.comm_reduction(r1, r2)


def test_native_local_search_swap_for_swap():
    """bs_local_search (C++/OpenMP, numpy's power kernel passed in) against
    the numpy restatement of placement.py:182-281 on random instances: the
    same final W and the same relaxed history bit for bit (so the same swap
    sequence), over p = 1, 2, 3, 4, inf, tied columns, LSA and random starts,
    and up to B = 128 patches (C5: 32 views x 2^2 patches, N = 8)."""
    rng = np.random.default_rng(2024)
    swaps = 0
    for trial in range(160):
        N = int(rng.choice([2, 3, 4, 8]))
        B = 128 if trial % 40 == 0 else N * int(rng.integers(1, 9))
        if B % N:
            B = N * (B // N)
        A = rng.integers(0, 10 ** int(rng.integers(2, 8)), size=(B, N))
        if trial % 3 == 0 and N > 1:
            A[:, 0] = A[:, 1]  # ties between candidate swaps
        p = float([1.0, 2.0, 3.0, 4.0, np.inf][trial % 5])
        co = asg.CostCoefficients(alpha=0.0, beta=float(rng.random()), gamma=float(rng.random()),
                                  delta=float(rng.random()) + 0.1, p=p)
        if trial % 2:
            init = asg.lsa_assign(A, B // N)
        else:
            init = asg.PlacementSolution(np.repeat(np.arange(N), B // N)[rng.permutation(B)], N)
        s1, i1 = asg.local_search(A, init, co, native=False)
        s2, i2 = asg.local_search(A, init, co, native=True)
        assert np.array_equal(s1.assignment, s2.assignment)
        assert i1["relaxed_history"] == i2["relaxed_history"]
        assert np.array_equal(init.assignment, s1.assignment) or i1["n_swaps"] > 0
        swaps += i1["n_swaps"]
    assert swaps > 500


def test_native_local_search_limits():
    """max_sweeps and errors: the native search stops after max_sweeps swaps
    like the numpy one, and rejects a W outside [0, N)."""
    rng = np.random.default_rng(5)
    A = rng.integers(0, 10**6, size=(64, 8))
    init = asg.PlacementSolution(np.repeat(np.arange(8), 8)[rng.permutation(64)], 8)
    for k in (0, 1, 3):
        s1, i1 = asg.local_search(A, init, INTER, max_sweeps=k, native=False)
        s2, i2 = asg.local_search(A, init, INTER, max_sweeps=k, native=True)
        assert i2["n_swaps"] == i1["n_swaps"] <= k and np.array_equal(s1.assignment, s2.assignment)
    from paper_2512_20017_b200 import _native as nat
    W = np.full(64, 9, dtype=np.int64)
    hist = np.empty(2)
    n = np.zeros(1, dtype=np.int64)
    with pytest.raises(asg.ParameterError):
        nat.host_call("bs_local_search", 64, 8, np.ascontiguousarray(A).ctypes.data, W.ctypes.data, 0.25, 0.25, 0.5,
                      4.0, 1, -1.0, None, 1, hist.ctypes.data, n.ctypes.data)
