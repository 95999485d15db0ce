"""The exchange-side kernels of the distributed step against numpy:
bs_canonical_order (canonical global-id order of received rows, SURVEY.md
§7(iii)), bs_gather_rows (any width), bs_return_rows (gradient rows back to
their owners' send-layout slots), bs_row_support (the rasterisers' per-row
support threshold vs the projection's own)."""

import numpy as np
import pytest
import torch

from paper_2512_20017_b200 import _native as nat

pytestmark = pytest.mark.gpu


def test_canonical_order_matches_numpy(cuda):
    rng = np.random.default_rng(0)
    # 3 sources x 4 slots; each segment ascending global ids (a source's rows of a view)
    seg_rows, seg_slot, gids = [], [], []
    for s in range(3):
        for slot in range(4):
            n = int(rng.integers(0, 500))
            ids = np.sort(rng.choice(2_000_000, n, replace=False)) + s  # may collide across sources: +s keeps unique
            seg_rows.append(n)
            seg_slot.append(slot)
            gids.append(ids)
    gid = np.concatenate(gids).astype(np.int32)
    n = len(gid)
    seg_row0 = np.concatenate([[0], np.cumsum(seg_rows)[:-1]]).astype(np.int64)
    slot_of_row = np.repeat(np.asarray(seg_slot), seg_rows)
    want = np.lexsort((gid, slot_of_row))
    g = torch.as_tensor(gid, device=cuda)
    order = torch.empty(n, dtype=torch.int64, device=cuda)
    cg = torch.empty(n, dtype=torch.int32, device=cuda)
    ws = torch.empty(nat.load().bs_canonical_order_workspace(n), dtype=torch.uint8, device=cuda)
    # device inputs held in locals: a temporary freed before the launch is
    # recycled by the caching allocator for the next argument
    r0_d = torch.as_tensor(seg_row0, device=cuda)
    sl_d = torch.as_tensor(np.asarray(seg_slot, dtype=np.int32), device=cuda)
    nat.call("bs_canonical_order", nat.ptr(g), n, nat.ptr(r0_d), nat.ptr(sl_d), len(seg_rows), 4,
             nat.ptr(order), nat.ptr(cg), nat.ptr(ws), ws.numel(), nat.stream_handle())
    assert np.array_equal(order.cpu().numpy(), want)
    assert np.array_equal(cg.cpu().numpy(), gid[want])


@pytest.mark.parametrize("width", [1, 3, 12, 24])
def test_gather_rows_any_width(cuda, width):
    rng = np.random.default_rng(width)
    src = rng.normal(size=(1000, width)).astype(np.float32)
    idx = rng.integers(0, 1000, 777).astype(np.int64)
    out = torch.empty((777, width), dtype=torch.float32, device=cuda)
    src_d, idx_d = torch.as_tensor(src, device=cuda), torch.as_tensor(idx, device=cuda)
    nat.call("bs_gather_rows", nat.ptr(src_d), width, nat.ptr(idx_d), 777, nat.ptr(out), nat.stream_handle())
    assert np.array_equal(out.cpu().numpy(), src[idx])


def test_return_rows_to_owner_slots(cuda):
    """Canonical row i came from received row order[i] of segment s = (source,
    view); its first `width` floats land at dst[source] + (seg_dst0[s] + k) rows."""
    rng = np.random.default_rng(1)
    n_src, width, src_w, dst_w = 3, 9, 12, 12
    seg_rows = [37, 0, 120, 5, 64, 18]
    seg_src = [0, 0, 1, 1, 2, 2]
    seg_dst0 = [0, 37, 3, 200, 10, 74]
    n = sum(seg_rows)
    seg_row0 = np.concatenate([[0], np.cumsum(seg_rows)[:-1]]).astype(np.int64)
    order = rng.permutation(n).astype(np.int64)
    src = rng.normal(size=(n, src_w)).astype(np.float32)
    homes = [torch.zeros((400, dst_w), dtype=torch.float32, device=cuda) for _ in range(n_src)]
    dst = torch.as_tensor(np.array([h.data_ptr() for h in homes], dtype=np.int64), device=cuda)
    keep = [torch.as_tensor(a, device=cuda) for a in (src, order, seg_row0, np.asarray(seg_src, dtype=np.int32),
                                                       np.asarray(seg_dst0, dtype=np.int64))]
    nat.call("bs_return_rows", nat.ptr(keep[0]), src_w, width, nat.ptr(keep[1]), n, nat.ptr(keep[2]),
             nat.ptr(keep[3]), nat.ptr(keep[4]), len(seg_rows), nat.ptr(dst), dst_w, nat.stream_handle())
    want = [np.zeros((400, dst_w), dtype=np.float32) for _ in range(n_src)]
    seg_of = np.repeat(np.arange(len(seg_rows)), seg_rows)
    for i in range(n):
        r = order[i]
        s = seg_of[r]
        want[seg_src[s]][seg_dst0[s] + r - seg_row0[s], :width] = src[i, :width]
    for h, w in zip(homes, want):
        assert np.array_equal(h.cpu().numpy(), w)


@pytest.mark.parametrize("model", ["3dgs", "2dgs"])
def test_row_support_equals_projection(cuda, model):
    """bs_row_support over received rows reproduces, bit for bit, the
    threshold the projection wrote with the rows (single-rank path)."""
    from paper_2512_20017_b200.trainer import SplatTrainer

    from _scene import c1_setup

    ds, params, gb, aabb, gt = c1_setup()
    tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, model=model)
    tr.step([0, 2, 5])
    torch.cuda.synchronize()
    n = tr.last["n_rows"]
    ref = tr.buf.bufs["row_support"][:n].clone()
    out = torch.empty(n, dtype=torch.float32, device=cuda)
    nat.call("bs_row_support", nat.ptr(tr.last["sp"]), tr.model_id, n, nat.ptr(out), nat.stream_handle())
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.cpu().numpy().view(np.uint32))
