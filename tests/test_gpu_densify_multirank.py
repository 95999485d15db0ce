"""Densification with the shard split over two ranks (sharing cuda:0, as in
tests/test_gpu_multirank.py) equals densification of the whole scene on one
rank: the same new points under the same renumbered global ids (groups in
global order, SplatTrainer._renumber), so the next training step's per-tile
lists of global ids and its images are bit-identical to the single rank's."""

import os

import numpy as np
import pytest
import torch

from test_gpu_multirank import BATCH, _gid_lists, _port, _setup

pytestmark = pytest.mark.gpu

CFG = dict(grad_threshold=2e-4, split_scale=0.5, min_opacity=0.05, seed=3)


def _stats_for(gid):
    """A deterministic statistic per global point id (every action occurs)."""
    h = (np.asarray(gid, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(40)
    u = (h % np.uint64(1000)).astype(np.float32) / 1000.0
    cnt = (1 + (h >> np.uint64(12)) % np.uint64(4)).astype(np.float32)
    return np.stack([cnt * u * 4e-4, cnt], axis=1).astype(np.float32)


def _low_opacity(params, gid):
    p = params.copy()
    p[0, (np.asarray(gid) % 11) == 0, 3] = -4.0  # ~9 % pruned
    return p


def _worker(rank, world, port, q, peer):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2512_20017_b200.exchange import PeerExchange, SplatExchange
    from paper_2512_20017_b200.sharding import build_bipartite_graph, hierarchical_partition
    from paper_2512_20017_b200.trainer import DensifyConfig, SplatTrainer

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ds, g, params, gt = _setup()
        params = _low_opacity(params, np.arange(params.shape[1]))
        part = hierarchical_partition(build_bipartite_graph(g, ds), world, 1, eps=0.05, seed=5)
        mine = np.flatnonzero(part.flat_gpus() == rank)
        pts = np.concatenate([np.arange(g.groups[k].begin, g.groups[k].end) for k in mine])
        gb = np.concatenate([[0], np.cumsum([g.groups[k].size for k in mine])]).astype(np.int32)
        tr = SplatTrainer(np.ascontiguousarray(params[:, pts, :]), gb, g.aabbs.reshape(-1, 6)[mine], ds.views,
                          gt=gt, comm=PeerExchange.create() if peer else SplatExchange(), global_ids=pts)
        tr.track_densify_stats(True)
        tr.densify_stats.copy_(torch.as_tensor(_stats_for(pts), device=tr.dev))
        rep = tr.densify(DensifyConfig(**CFG))
        gid = tr.global_ids.cpu().numpy()
        dens = tr.params.cpu().numpy()
        tr.step(BATCH)
        n = len(tr.last["layout"].my_views)
        img = tr.last["image"][: n * 96 * 160 * 3].cpu().numpy().reshape(n, 96, 160, 3) if n else None
        q.put((rank, gid, dens, [BATCH[v] for v in tr.last["layout"].my_views], img,
               _gid_lists(tr, n) if n else None, rep["n_after"]))
        if peer:
            tr.comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("peer", [False, True])
def test_two_rank_densify_matches_single_rank(cuda, peer):
    import torch.multiprocessing as mp

    from paper_2512_20017_b200.trainer import DensifyConfig, SplatTrainer

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, peer)) for r in range(2)]
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
    params = _low_opacity(params, np.arange(params.shape[1]))
    tr = SplatTrainer(params, g.group_begin(), g.aabbs.reshape(-1, 6), ds.views, gt=gt)
    tr.record_row_gid = True
    tr.track_densify_stats(True)
    tr.densify_stats.copy_(torch.as_tensor(_stats_for(np.arange(params.shape[1])), device=tr.dev))
    rep = tr.densify(DensifyConfig(**CFG))
    assert rep["cloned"] > 0 and rep["split"] > 0 and rep["pruned"] > 0
    after = tr.params.cpu().numpy()
    # the ranks' new points, under their new global ids, are the single rank's points bit for bit
    ids = np.concatenate([res[0][1], res[1][1]])
    assert res[0][6] + res[1][6] == tr.S and np.array_equal(np.sort(ids), np.arange(tr.S))
    for r in (0, 1):
        assert np.all(np.diff(res[r][1]) > 0)
        assert np.array_equal(res[r][2].view(np.uint32), after[:, res[r][1], :].view(np.uint32))
    tr.step(BATCH)
    lists_ref = _gid_lists(tr, len(BATCH))
    img_ref = tr.last["image"][: len(BATCH) * 96 * 160 * 3].cpu().numpy().reshape(len(BATCH), 96, 160, 3)
    assert sorted(res[0][3] + res[1][3]) == sorted(BATCH)
    for r in (0, 1):
        for slot, v in enumerate(res[r][3]):
            k = BATCH.index(v)
            for t, (a, b) in enumerate(zip(res[r][5][slot], lists_ref[k])):
                assert np.array_equal(a, b), f"view {v} tile {t}"
            assert np.array_equal(res[r][4][slot], img_ref[k]), f"view {v}"
