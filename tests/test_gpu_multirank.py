"""Two ranks of the full GPU training step (SplatTrainer + SplatExchange)
sharing cuda:0 over gloo (host-staged all-to-all), against the single-rank
step on the whole scene: every rendered view and every updated parameter
must agree (the points-to-rank partition is the paper's offline placement,
the image-to-rank assignment hierarchical_place on the all-gathered A)."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

BATCH = [0, 2, 5, 7]
BATCH2 = [1, 3, 4, 6]


def _setup():
    from paper_2512_20017_b200 import scenes
    from paper_2512_20017_b200.culling import zorder_group

    ds = scenes.generate_aerial_scene(0, 20_000, (1, 2), 8, 50.0, (160, 96))
    g = zorder_group(ds.cloud, G=256)
    params = scenes.init_gaussians(g.sorted_cloud, 0, scenes.mean_spacing(50.0, (1, 2), 20_000))
    gt = scenes.synthetic_gt(0, 8, 160, 96)
    return ds, g, params, gt


def _worker(rank, world, port, q, prefetch=False, patches=1, peer=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2512_20017_b200 import scenes
    from paper_2512_20017_b200.exchange import PeerExchange, SplatExchange
    from paper_2512_20017_b200.sharding import build_bipartite_graph, hierarchical_partition
    from paper_2512_20017_b200.trainer import AdamConfig, SplatTrainer

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ds, g, params, gt = _setup()
        part = hierarchical_partition(build_bipartite_graph(g, ds), world, 1, eps=0.05, seed=5)
        mine = np.flatnonzero(part.flat_gpus() == rank)
        pts = np.concatenate([np.arange(g.groups[k].begin, g.groups[k].end) for k in mine])
        sizes = [g.groups[k].size for k in mine]
        gb = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
        tr = SplatTrainer(np.ascontiguousarray(params[:, pts, :]), gb, g.aabbs.reshape(-1, 6)[mine], ds.views,
                          gt=gt, adam=AdamConfig(scenes.lr_table(50.0)),
                          comm=PeerExchange.create() if peer else SplatExchange(), patches=patches,
                          global_ids=pts)
        if peer:
            assert getattr(tr.comm, "peer", False), "peer exchange preflight failed"
        if prefetch:
            # step 1 starts the asynchronous placement of step 2 (stale W)
            tr.step(BATCH, next_batch=BATCH2)
            losses = tr.step(BATCH2).cpu().numpy()
            assert tr.comm.prefetched == 1
            batch = BATCH2
        else:
            losses = tr.step(BATCH).cpu().numpy()
            batch = BATCH
        my_views = tr.last["layout"].my_views if patches == 1 else tr.last["my_views"]
        n = len(my_views)
        img = tr.last["image"][: n * 96 * 160 * 3].cpu().numpy().reshape(n, 96, 160, 3) if n else None
        q.put((rank, pts, tr.params.cpu().numpy(), [batch[v] for v in my_views], img, losses,
               tr.last["A"], tr.last["W"], _gid_lists(tr, n) if n else None, tr.comm.bytes_fwd))
        if peer:
            tr.comm.close()
    finally:
        dist.destroy_process_group()


def _gid_lists(tr, n_slots):
    """Per rendered slot and tile: the global ids of the tile's depth-sorted
    instance list (rows mapped through the canonical row -> global id)."""
    T = tr.tiles
    rg = tr.last["ranges"][: n_slots * T * 2].cpu().numpy().reshape(n_slots, T, 2)
    irows = tr.last["irows"][: tr.last["n_inst"]].cpu().numpy().astype(np.int64)
    gid = tr.last["row_gid"].cpu().numpy()
    out = []
    for s in range(n_slots):
        out.append([gid[irows[a:b]] if b > a else np.zeros(0, np.int32) for a, b in rg[s]])
    return out


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("prefetch,peer", [(False, False), (True, False), (False, True), (True, True)])
def test_two_ranks_match_single_rank(cuda, prefetch, peer):
    """peer=True: the splat rows and their gradients move through CUDA IPC
    peer memory (exchange.PeerExchange: the projection writes into the
    renderer's buffer, bs_return_rows into the owner's, stream-ordered flags)
    instead of torch.distributed all-to-alls -- both ranks share cuda:0 here,
    the same loads/stores go over NVLink between GPUs."""
    import torch.multiprocessing as mp

    from paper_2512_20017_b200 import scenes
    from paper_2512_20017_b200.trainer import AdamConfig, SplatTrainer

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, prefetch, 1, peer)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        item = q.get(timeout=600)
        res[item[0]] = item
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single rank over the whole scene
    ds, g, params, gt = _setup()
    lr = scenes.lr_table(50.0)
    tr = SplatTrainer(params, g.group_begin(), g.aabbs.reshape(-1, 6), ds.views, gt=gt, adam=AdamConfig(lr))
    tr.record_row_gid = True
    if prefetch:
        tr.step(BATCH)
    batch = BATCH2 if prefetch else BATCH
    losses = tr.step(batch).cpu().numpy()
    lists_ref = _gid_lists(tr, len(batch))
    img_ref = tr.last["image"][: len(batch) * 96 * 160 * 3].cpu().numpy().reshape(len(batch), 96, 160, 3)
    after_ref = tr.params.cpu().numpy()
    A = res[0][6]
    assert np.array_equal(A, res[1][6]) and np.array_equal(res[0][7], res[1][7])
    assert np.array_equal(A.sum(axis=1), tr.last["rows_per_view"])  # the same visible sets
    assert sorted(res[0][3] + res[1][3]) == sorted(batch)
    for r in (0, 1):
        for slot, v in enumerate(res[r][3]):
            k = batch.index(v)
            if not prefetch:
                # canonical order (bs_canonical_order): the per-tile lists of
                # global ids are the single-rank lists bit for bit, and so the
                # forward image is bit-identical
                for t, (a, b) in enumerate(zip(res[r][8][slot], lists_ref[k])):
                    assert np.array_equal(a, b), f"view {v} tile {t}"
                assert np.array_equal(res[r][4][slot], img_ref[k]), f"view {v}"
                assert res[r][5][slot] == losses[k]
            else:
                # second step: parameters after step 1 agree to the Adam
                # tolerance below, so the images to the parity tolerance
                assert np.abs(res[r][4][slot] - img_ref[k]).max() <= 1e-4, f"view {v}"
                assert abs(res[r][5][slot] - losses[k]) <= 1e-4
        pts, after = res[r][1], res[r][2]
        ref = after_ref[:, pts, :]
        lr_full = np.broadcast_to(lr.reshape(15, 1, 4), ref.shape)
        diff = np.abs(after - ref)
        steps = 2 if prefetch else 1
        assert (diff <= 1e-3 * lr_full + 1e-7).mean() > (0.99 if prefetch else 0.999)
        assert (diff <= 2.0 * steps * lr_full + 1e-6).all()


def test_two_ranks_patches_match_single_rank(cuda):
    """P = 2: the 4 x 4 = 16 patches of the batch are placed on 2 ranks; each
    rank renders only its patches from the splats whose support reaches them
    (csrc/patches.cu); the assembled images equal the single-rank render."""
    import torch.multiprocessing as mp

    from paper_2512_20017_b200 import scenes
    from paper_2512_20017_b200.trainer import AdamConfig, SplatTrainer

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, False, 2)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        item = q.get(timeout=600)
        res[item[0]] = item
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ds, g, params, gt = _setup()
    lr = scenes.lr_table(50.0)
    tr = SplatTrainer(params, g.group_begin(), g.aabbs.reshape(-1, 6), ds.views, gt=gt, adam=AdamConfig(lr))
    losses = tr.step(BATCH).cpu().numpy()
    img_ref = tr.last["image"][: len(BATCH) * 96 * 160 * 3].cpu().numpy().reshape(len(BATCH), 96, 160, 3)
    after_ref = tr.params.cpu().numpy()
    A, W = res[0][6], res[0][7]
    assert A.shape == (len(BATCH) * 4, 2) and np.array_equal(W, res[1][7])
    assert np.bincount(W, minlength=2).tolist() == [8, 8]
    # per view: assemble the patches from their renderers
    P, Wimg, Himg = 2, 160, 96
    xs = [(c * Wimg) // P for c in range(P + 1)]
    ys = [(r * Himg) // P for r in range(P + 1)]
    loss_sum = np.zeros(len(BATCH))
    for k, v in enumerate(BATCH):
        img = np.full((Himg, Wimg, 3), np.nan, dtype=np.float32)
        for j in range(P * P):
            r_, c_ = divmod(j, P)
            owner = int(W[k * P * P + j])
            slot = res[owner][3].index(v)
            img[ys[r_]:ys[r_ + 1], xs[c_]:xs[c_ + 1]] = res[owner][4][slot][ys[r_]:ys[r_ + 1], xs[c_]:xs[c_ + 1]]
        assert np.array_equal(img, img_ref[k]), f"view {v}"  # canonical order: bit-identical
        for r in (0, 1):
            if v in res[r][3]:
                loss_sum[k] += res[r][5][res[r][3].index(v)]
    np.testing.assert_allclose(loss_sum, losses, rtol=0, atol=1e-6)  # patch losses add up to the view's
    for r in (0, 1):
        pts, after = res[r][1], res[r][2]
        ref = after_ref[:, pts, :]
        lr_full = np.broadcast_to(lr.reshape(15, 1, 4), ref.shape)
        diff = np.abs(after - ref)
        assert (diff <= 1e-3 * lr_full + 1e-7).mean() > 0.999
        assert (diff <= 2.0 * lr_full + 1e-6).all()


def _c2_worker(rank, world, port, q):
    """One rank of the C2 configuration (1M Gaussians, 1080p, batch 4) over
    the peer-memory exchange."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2512_20017_b200 import scenes
    from paper_2512_20017_b200.culling import zorder_group
    from paper_2512_20017_b200.exchange import PeerExchange
    from paper_2512_20017_b200.sharding import build_bipartite_graph, hierarchical_partition
    from paper_2512_20017_b200.trainer import AdamConfig, SplatTrainer

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ds = scenes.generate_aerial_scene(1, 1_000_000, (1, 1), 8, 50.0, (1920, 1080))
        g = zorder_group(ds.cloud, G=2048)
        part = hierarchical_partition(build_bipartite_graph(g, ds), world, 1, eps=0.05, seed=5)
        mine = np.flatnonzero(part.flat_gpus() == rank)
        pts = np.concatenate([np.arange(g.groups[k].begin, g.groups[k].end) for k in mine])
        gb = np.concatenate([[0], np.cumsum([g.groups[k].size for k in mine])]).astype(np.int32)
        params = scenes.init_gaussians_rows(g.sorted_cloud, 1, scenes.mean_spacing(50.0, (1, 1), 1_000_000), pts)
        gt = scenes.synthetic_gt(1, 8, 1920, 1080)
        tr = SplatTrainer(params, gb, g.aabbs.reshape(-1, 6)[mine], ds.views, gt=gt,
                          adam=AdamConfig(scenes.lr_table(50.0)), comm=PeerExchange.create(), global_ids=pts)
        assert getattr(tr.comm, "peer", False)
        tr.step(C2_BATCH)
        torch.cuda.synchronize()
        views = [C2_BATCH[v] for v in tr.last["layout"].my_views]
        n = len(views)
        T = tr.tiles
        rg = tr.last["ranges"][: n * T * 2].cpu().numpy().reshape(n, T, 2)
        irows = tr.last["irows"][: tr.last["n_inst"]].cpu().numpy().astype(np.int64)
        gid = tr.last["row_gid"].cpu().numpy()
        lists = [(rg[s, :, 1] - rg[s, :, 0], np.concatenate([gid[irows[a:b]] for a, b in rg[s] if b > a]))
                 for s in range(n)]
        img = tr.last["image"][: n * 1080 * 1920 * 3].cpu().numpy().reshape(n, 1080, 1920, 3)
        q.put((rank, views, lists, img, tr.comm.bytes_fwd))
        tr.comm.close()
    finally:
        dist.destroy_process_group()


C2_BATCH = [0, 3, 4, 7]


def test_two_ranks_c2_scale_lists_bit_identical(cuda):
    """BASELINE configs[1] size (1M Gaussians, 1080p, batch 4) on 2 ranks over
    the peer exchange: every rendered view's per-tile lists (as global point
    ids) and its image are bit-identical to the single-rank step's -- the
    canonical order at the scale the throughput is quoted on."""
    import torch.multiprocessing as mp

    from paper_2512_20017_b200 import scenes
    from paper_2512_20017_b200.culling import zorder_group
    from paper_2512_20017_b200.trainer import SplatTrainer

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_c2_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        item = q.get(timeout=900)
        res[item[0]] = item
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ds = scenes.generate_aerial_scene(1, 1_000_000, (1, 1), 8, 50.0, (1920, 1080))
    g = zorder_group(ds.cloud, G=2048)
    params = scenes.init_gaussians(g.sorted_cloud, 1, scenes.mean_spacing(50.0, (1, 1), 1_000_000))
    gt = scenes.synthetic_gt(1, 8, 1920, 1080)
    tr = SplatTrainer(params, g.group_begin(), g.aabbs.reshape(-1, 6), ds.views, gt=gt)
    tr.record_row_gid = True
    tr.step(C2_BATCH)
    torch.cuda.synchronize()
    T = tr.tiles
    rg = tr.last["ranges"][: 4 * T * 2].cpu().numpy().reshape(4, T, 2)
    irows = tr.last["irows"][: tr.last["n_inst"]].cpu().numpy().astype(np.int64)
    gid = tr.last["row_gid"].cpu().numpy()
    img = tr.last["image"][: 4 * 1080 * 1920 * 3].cpu().numpy().reshape(4, 1080, 1920, 3)
    seen = []
    for r in (0, 1):
        assert res[r][4] > 0  # rows really crossed between the ranks
        for slot, v in enumerate(res[r][1]):
            k = C2_BATCH.index(v)
            lens, flat = res[r][2][slot]
            assert np.array_equal(lens, rg[k, :, 1] - rg[k, :, 0]), f"view {v}: list lengths"
            ref = np.concatenate([gid[irows[a:b]] for a, b in rg[k] if b > a])
            assert np.array_equal(flat, ref), f"view {v}: per-tile lists"
            assert np.array_equal(res[r][3][slot], img[k]), f"view {v}: image"
            seen.append(v)
    assert sorted(seen) == sorted(C2_BATCH)


def test_four_ranks_peer_match_single_rank(cuda):
    """4 ranks (one view each) over the peer-memory exchange: per-tile lists of
    global ids and images bit-identical to the single-rank step."""
    import torch.multiprocessing as mp

    from paper_2512_20017_b200.trainer import SplatTrainer

    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, False, 1, True)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        item = q.get(timeout=600)
        res[item[0]] = item
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ds, g, params, gt = _setup()
    tr = SplatTrainer(params, g.group_begin(), g.aabbs.reshape(-1, 6), ds.views, gt=gt)
    tr.record_row_gid = True
    tr.step(BATCH)
    lists_ref = _gid_lists(tr, len(BATCH))
    img_ref = tr.last["image"][: len(BATCH) * 96 * 160 * 3].cpu().numpy().reshape(len(BATCH), 96, 160, 3)
    seen = []
    for r in range(world):
        assert np.array_equal(res[r][6], res[0][6]) and np.array_equal(res[r][7], res[0][7])
        for slot, v in enumerate(res[r][3]):
            k = BATCH.index(v)
            for t, (a, b) in enumerate(zip(res[r][8][slot], lists_ref[k])):
                assert np.array_equal(a, b), f"rank {r} view {v} tile {t}"
            assert np.array_equal(res[r][4][slot], img_ref[k]), f"rank {r} view {v}"
            seen.append(v)
    assert sorted(seen) == sorted(BATCH)
