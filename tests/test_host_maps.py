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
    sol, info = asg.local_search(mat, asg.lsa_assign(mat, B // N), asg.CostCoefficients())
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
