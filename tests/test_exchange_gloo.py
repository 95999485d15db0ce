"""world_size-2 gloo test of the distributed step's plumbing on CPU
(exchange.py): all-gather of C[v]_k into A, W = hierarchical_place(A),
send/recv layouts, the SP all-to-all and the reverse G_SP all-to-all.

Each rank holds half of the Z-ordered point groups.  The per-view compute
(projection, render, backward) is done here by the CPU oracle as TEST
SCAFFOLDING (the product runs those on the GPU); what is under test is that
the exchanged rows reproduce, bit for bit, the single-process result: the
rendered images of every view, the per-point gradients, and the
A-predicted transfer volumes of account_iteration.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import py_oracle
from paper_2512_20017_b200 import scenes
from paper_2512_20017_b200.accounting import ClusterTopology, account_iteration
from paper_2512_20017_b200.assign import PlacementSolution
from paper_2512_20017_b200.culling import batch_planes
from paper_2512_20017_b200.exchange import SplatExchange, layout_for
from paper_2512_20017_b200.trainer import camera_bytes

W_IMG, H_IMG = 64, 48


def _scene():
    ds = scenes.generate_aerial_scene(2, 3000, (1, 2), 4, 20.0, (W_IMG, H_IMG))
    perm, gb, aabb = py_oracle.zorder_layout(ds.cloud.positions, 64)
    sorted_cloud = scenes.PointCloud(ds.cloud.positions[perm])
    params = scenes.init_gaussians(sorted_cloud, 2, scenes.mean_spacing(20.0, (1, 2), 3000))
    gt = scenes.synthetic_gt(2, 4, W_IMG, H_IMG)
    return ds, params, gb, aabb, gt


def _shard(gb, rank, world):
    ng = len(gb) - 1
    lo, hi = (ng * rank) // world, (ng * (rank + 1)) // world
    return np.arange(gb[lo], gb[hi]), gb[lo:hi + 1] - gb[lo], lo, hi


def _render_view(sp_rows, gt_img):
    img, T, nc = py_oracle.render(sp_rows, W_IMG, H_IMG)
    loss, gimg = py_oracle.l1_loss(img, gt_img)
    gsp = py_oracle.render_bwd(sp_rows, W_IMG, H_IMG, T, nc, gimg)
    return img, loss, gsp


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ds, params, gb, aabb, gt = _scene()
        views = ds.views
        pts, lgb, lo, hi = _shard(gb, rank, world)
        local = np.ascontiguousarray(params[:, pts, :])
        planes = batch_planes(views, 1)
        mask = py_oracle.visibility_mask(local[0, :, :3], lgb, aabb[lo:hi], planes, len(views))
        col = torch.tensor([int(((mask >> v) & 1).sum()) for v in range(len(views))], dtype=torch.int64)
        ex = SplatExchange()
        A = ex.gather_access(col)
        Wv = ex.assign(A)
        lay = layout_for(A, Wv, rank)
        # send buffer: views in destination order, local rows ascending
        send, idx_of = [], {}
        for v in lay.order:
            idx = np.flatnonzero((mask >> v) & 1).astype(np.int64)
            idx_of[int(v)] = idx
            send.append(py_oracle.project(local, idx, camera_bytes([views[v]]), 3))
        send = torch.as_tensor(np.concatenate(send)) if send else torch.zeros((0, 12))
        recv = ex.forward(send.reshape(-1), lay, 12).numpy()
        # render my views from the received segments
        offs = np.concatenate([[0], np.cumsum(lay.seg_rows)])
        g_recv = np.zeros((lay.n_recv, 9), dtype=np.float32)
        images = {}
        for slot, v in enumerate(lay.my_views):
            segs = [k for k in range(len(lay.seg_slot)) if lay.seg_slot[k] == slot]
            rows = np.concatenate([np.arange(offs[k], offs[k + 1]) for k in segs])
            img, loss, gsp = _render_view(recv[rows], gt[v])
            images[int(v)] = (img, loss)
            g_recv[rows] = gsp
        g_send = ex.backward(torch.as_tensor(g_recv).reshape(-1), lay, 9).numpy()
        # projection backward of the local shard from the returned rows
        grad = np.zeros_like(local)
        r = 0
        for v in lay.order:
            idx = idx_of[int(v)]
            py_oracle.project_bwd(local, idx, camera_bytes([views[v]]), 3, g_send[r:r + len(idx)], grad)
            r += len(idx)
        out_q.put((rank, A, Wv, images, pts, grad, ex.bytes_fwd, ex.bytes_bwd))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_exchange_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        item = q.get(timeout=300)
        res[item[0]] = item
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference: every view from all points (ascending global id)
    ds, params, gb, aabb, gt = _scene()
    planes = batch_planes(ds.views, 1)
    mask = py_oracle.visibility_mask(params[0, :, :3], gb, aabb, planes, len(ds.views))
    grad_ref = np.zeros_like(params)
    A = res[0][1]
    assert np.array_equal(A, res[1][1]) and np.array_equal(res[0][2], res[1][2])
    W = res[0][2]
    for v, view in enumerate(ds.views):
        idx = np.flatnonzero((mask >> v) & 1).astype(np.int64)
        assert A[v].sum() == len(idx)
        sp = py_oracle.project(params, idx, camera_bytes([view]), 3)
        img, loss, gsp = _render_view(sp, gt[v])
        owner = int(W[v])
        got_img, got_loss = res[owner][3][v]
        assert np.array_equal(got_img, img), f"view {v}"
        assert got_loss == loss
        py_oracle.project_bwd(params, idx, camera_bytes([view]), 3, gsp, grad_ref)
    for r in range(world):
        pts, grad = res[r][4], res[r][5]
        np.testing.assert_allclose(grad, grad_ref[:, pts, :], rtol=0, atol=1e-9)
    # moved rows == A-predicted transfers (ClusterTopology(N, 1), P = 1)
    tr = account_iteration(A, PlacementSolution(W, world), ClusterTopology(world, 1, 1e9, 1e9), 48)
    assert sum(res[r][6] for r in range(world)) == int(tr.send_inter.sum()) * 48
    assert sum(res[r][7] for r in range(world)) == int(tr.recv_inter.sum()) * 36


def _prefetch_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = SplatExchange()
        rng = np.random.default_rng(100 + rank)
        stale = torch.as_tensor(rng.integers(0, 5000, 8), dtype=torch.int64)
        fresh = stale + torch.as_tensor(rng.integers(0, 50, 8), dtype=torch.int64)
        ex.prefetch(stale, key=(1, 2, 3, 4, 5, 6, 7, 8))      # issued during step t
        A = ex.gather_access(fresh)                          # step t+1: fresh counts
        W = ex.assign(A, key=(1, 2, 3, 4, 5, 6, 7, 8))        # the prefetched (stale) W
        A_stale = torch.empty(world * 8, dtype=torch.int64)
        dist.all_gather_into_tensor(A_stale, stale)
        out_q.put((rank, A, W, A_stale.view(world, -1).t().numpy(), ex.prefetched, ex.assign(A, key=None)))
    finally:
        dist.destroy_process_group()


def test_two_rank_async_placement():
    """prefetch(): the W of the next batch is computed on a host thread from
    the stale all-gathered counts; identical on every rank."""
    from paper_2512_20017_b200.assign import CostCoefficients, hierarchical_place

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_prefetch_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        item = q.get(timeout=300)
        res[item[0]] = item
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, A, W, A_stale, n_pref, W_fresh = res[0]
    assert n_pref == 1
    assert np.array_equal(W, res[1][2]) and np.array_equal(A, res[1][1])
    inter = CostCoefficients(p=4.0)
    intra = CostCoefficients(alpha=0.0, beta=0.1, gamma=0.1, delta=1.0, p=4.0)
    assert np.array_equal(W, hierarchical_place(A_stale, world, 1, inter, intra).assignment)
    assert np.array_equal(W_fresh, hierarchical_place(A, world, 1, inter, intra).assignment)
    assert np.bincount(W, minlength=world).tolist() == [4, 4]
