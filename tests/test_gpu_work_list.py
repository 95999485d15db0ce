"""Visible-chunk work list (bs_cull_desc.work_list -> bs_proj_desc.work_list):
the projection and the selective fused Adam visit only the 256-point chunks
the culling listed, in no particular order.  Rows are placed by the chunk
prefixes and points update independently, so a step with the list equals a
step without it bit for bit: splat rows, per-tile lists, image, losses and
after the update the parameters to the Adam tolerance (G_SP is accumulated
by atomics in both runs); with selective Adam the hidden points stay
untouched (3DGS and 2DGS, one- and multi-chunk groups)."""

import numpy as np
import pytest
import torch

from paper_2512_20017_b200 import scenes
from paper_2512_20017_b200.trainer import AdamConfig, SplatTrainer

from _scene import c1_setup

pytestmark = pytest.mark.gpu


def _run(on, model, selective, G, batch):
    ds, params, gb, aabb, gt = c1_setup(G=G)
    lr = scenes.lr_table(50.0)
    tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, model=model, adam=AdamConfig(lr, selective=selective))
    tr.visible_chunk_list = on
    losses = tr.step(batch).cpu().numpy()
    n, ni = tr.last["n_rows"], tr.last["n_inst"]
    fwd = (losses, tr.last["sp"][: n * tr.sp_floats].cpu().numpy(), tr.last["irows"][:ni].cpu().numpy(),
           tr.last["image"].cpu().numpy())
    torch.cuda.synchronize()
    mask = tr.buf.bufs["mask"][: tr.S].cpu().numpy()
    return fwd, tr.params.cpu().numpy(), tr.exp_avg.cpu().numpy(), params, mask, lr


@pytest.mark.parametrize("model", ["3dgs", "2dgs"])
@pytest.mark.parametrize("selective", [False, True])
@pytest.mark.parametrize("G", [256, 1000])
@pytest.mark.parametrize("batch", [[0, 3], [1, 2, 6, 7]])
def test_work_list_matches_one_cta_per_chunk(cuda, model, selective, G, batch):
    a = _run(True, model, selective, G, batch)
    b = _run(False, model, selective, G, batch)
    # forward: bit for bit (rows placed by the chunk prefixes)
    for x, y in zip(a[0], b[0]):
        assert np.array_equal(x, y)
    # the update: G_SP is accumulated by atomics in either run, so the
    # parameters agree to the Adam tolerance of the multi-rank tests
    lr_full = np.broadcast_to(a[5].reshape(15, 1, 4), a[1].shape)
    diff = np.abs(a[1] - b[1])
    assert (diff <= 1e-3 * lr_full + 1e-7).mean() > 0.999
    assert (diff <= 2.0 * lr_full + 1e-6).all()
    if selective:  # points outside every batch view: parameters and moments untouched in both runs
        hidden = a[4] == 0
        assert hidden.any()
        for p_after, m_after in ((a[1], a[2]), (b[1], b[2])):
            assert np.array_equal(p_after[:, hidden], a[3][:, hidden])
            assert not m_after[:, hidden].any()


def test_list_chunks_matches_counts(cuda):
    """bs_list_chunks: exactly the (group, chunk) pairs whose chunk holds a
    point visible in some view, from the culling's counts / chunk prefixes."""
    ds, params, gb, aabb, gt = c1_setup(G=1000)
    tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt)
    tr.visible_chunk_list = True
    tr.step([0, 5])
    torch.cuda.synchronize()
    mask = tr.buf.bufs["mask"][: tr.S].cpu().numpy()
    gbh = np.asarray(gb, dtype=np.int64)
    want = set()
    for g in range(len(gbh) - 1):
        for c in range(tr.max_chunks):
            lo, hi = gbh[g] + 256 * c, min(gbh[g + 1], gbh[g] + 256 * (c + 1))
            if lo < hi and mask[lo:hi].any():
                want.add(g * tr.max_chunks + c)
    n = int(tr.buf.bufs["work_count"].cpu().numpy()[0])
    got = tr.buf.bufs["work_list"][:n].cpu().numpy()
    assert len(got) == len(set(got.tolist())) and set(got.tolist()) == want


def test_select_rows_and_copy_to_host(cuda):
    """bs_select_rows (view ids as kernel parameters), bs_upload (a host array
    as kernel parameters) and bs_copy_to_host (a kernel store into mapped
    pinned memory) against torch."""
    from paper_2512_20017_b200 import _native as nat

    table = torch.arange(40 * 7, dtype=torch.float32, device="cuda").reshape(40, 7)
    ids = np.array([3, 39, 0, 3, 17], dtype=np.int32)
    out = torch.empty((5, 7), dtype=torch.float32, device="cuda")
    nat.call("bs_select_rows", ids.ctypes.data, 5, nat.ptr(table), 40, 28, nat.ptr(out), nat.stream_handle())
    assert torch.equal(out, table[torch.as_tensor(ids.astype(np.int64), device="cuda")])
    with pytest.raises(Exception):
        bad = np.array([40], dtype=np.int32)
        nat.call("bs_select_rows", bad.ctypes.data, 1, nat.ptr(table), 40, 28, nat.ptr(out), nat.stream_handle())
    src = torch.arange(9, dtype=torch.int64, device="cuda") * 1000003
    pin = torch.zeros(9, dtype=torch.int64, pin_memory=True)
    nat.call("bs_copy_to_host", nat.ptr(src), 72, pin.data_ptr(), nat.stream_handle())
    torch.cuda.synchronize()
    assert torch.equal(pin, src.cpu())
    host = (np.arange(1300, dtype=np.int64) * 7919) % 104729  # > one 2 KB kernel-parameter chunk
    dev = torch.full((1300,), -1, dtype=torch.int64, device="cuda")
    nat.upload(host, dev)
    assert np.array_equal(dev.cpu().numpy(), host)
    with pytest.raises(Exception):  # pageable host memory is refused
        nat.call("bs_copy_to_host", nat.ptr(src), 72, torch.zeros(9, dtype=torch.int64).data_ptr(),
                 nat.stream_handle())
