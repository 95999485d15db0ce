"""The product's fused projection backward + Adam (bs_project_bwd_adam, the
kernel every training step runs) pinned beyond Adam step 1.

At Adam step 1 the update is lr * g / (|g| + eps) = lr * sign(g), so a
gradient with the right sign and a wrong magnitude passes a parameter
comparison.  Here the moments start non-zero (m ~ g scale, v ~ g^2 scale) and
the step counter is 3, so the new first moment m' = b1 m + (1 - b1) g carries
the gradient's magnitude: the gradient the kernel used is recovered from m'
and compared with the oracle's analytic gradient (oracle/splat_oracle.c,
project_bwd, which tests/test_oracle_cpu.py checks against float64 autograd)
at the suite's 1e-4 x per-(plane, lane) max tolerance; v' and the parameters
are compared with the oracle's Adam (torch.optim.Adam
semantics).  This covers the kernel's own staging: SH coefficients copied into
shared-memory columns (cp.async), SH gradients accumulated in shared-memory
columns, and the plane-batched Adam loop, for groups of one and of several
256-point chunks, dense and selective Adam, 3DGS and 2DGS.
"""

import numpy as np
import pytest
import torch

from paper_2512_20017_b200 import _native as nat
from paper_2512_20017_b200 import scenes
from paper_2512_20017_b200.trainer import AdamConfig, SplatTrainer, camera_bytes

from _scene import c1_setup

pytestmark = pytest.mark.gpu

GRAD_REL = 1e-4
B1, B2, EPS = 0.9, 0.999, 1e-15


def _layout(tr, batch, cuda):
    """Culling mask + per-(group, view) row bases of `batch` (as the step does)."""
    st = nat.stream_handle()
    B = len(batch)
    bt = torch.as_tensor(batch, device=cuda)
    planes = tr.planes_all.index_select(0, bt).contiguous()
    cams = tr.cams_all.index_select(0, bt).contiguous()
    mask = torch.empty(tr.S, dtype=torch.int32, device=cuda)
    counts = torch.empty(tr.n_groups * B, dtype=torch.int32, device=cuda)
    pre = torch.zeros(tr.n_groups * tr.max_chunks * B, dtype=torch.int32, device=cuda)
    nat.call("bs_cull_count", nat.CullDesc(nat.CULL_MASK, B, 1, 1, 0, 4, tr.max_chunks, nat.ptr(pre)),
             nat.ptr(tr.params), tr.S, None, nat.ptr(tr.group_begin), nat.ptr(tr.aabb), tr.n_groups, nat.ptr(planes),
             None, None, nat.ptr(mask), nat.ptr(counts), None, st)
    base = torch.empty_like(counts)
    vr = torch.empty(B, dtype=torch.int64, device=cuda)
    v0 = torch.empty(B, dtype=torch.int64, device=cuda)
    nat.call("bs_scan_counts", nat.ptr(counts), tr.n_groups, B, None, nat.ptr(base), nat.ptr(vr), nat.ptr(v0), st)
    return cams, mask, base, vr, v0, pre


@pytest.mark.parametrize("model,G,selective", [("3dgs", 256, 0), ("3dgs", 1000, 0), ("3dgs", 256, 1),
                                               ("2dgs", 256, 0), ("2dgs", 1000, 1)])
def test_fused_project_bwd_adam_step3(cuda, model, G, selective):
    from oracle import py_oracle

    ds, params, gb, aabb, gt = c1_setup(G=G)
    tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, sh_degree=3, model=model)
    batch = [2, 4, 7]
    B = len(batch)
    cams, mask, base, vr, v0, pre = _layout(tr, batch, cuda)
    n = int(vr.sum().item())
    wire, gsp_floats = (15, nat.GSP2_FLOATS) if model == "2dgs" else (9, nat.GSP_FLOATS)
    rng = np.random.default_rng(7 + G + selective)
    gw = rng.normal(0, 1e-3, (n, wire)).astype(np.float32)
    gsp = torch.zeros((n, gsp_floats), dtype=torch.float32, device=cuda)
    gsp[:, :wire] = torch.as_tensor(gw, device=cuda)
    # oracle gradient of the same G_SP rows (moments form), view by view
    m_host = mask.cpu().numpy().view(np.uint32)
    g_ref = np.zeros_like(params)
    row = 0
    for s, v in enumerate(batch):
        idx = np.flatnonzero((m_host >> s) & 1).astype(np.int64)
        py_oracle.project_bwd(params, idx, camera_bytes([ds.views[v]]), 3, gw[row:row + len(idx)], g_ref,
                              model=model)
        row += len(idx)
    assert row == n
    # non-zero moments at the gradient's scale, per (plane, lane)
    scale = np.abs(g_ref).reshape(15, -1, 4).max(axis=1, keepdims=True) + 1e-30  # [15, 1, 4]
    m0 = (rng.normal(0, 1, params.shape) * scale).astype(np.float32)
    v0h = (rng.uniform(0.5, 2.0, params.shape) * scale * scale).astype(np.float32)
    lr = scenes.lr_table(50.0)
    step = 3
    p_d = torch.as_tensor(params, device=cuda).clone()
    m_d = torch.as_tensor(m0, device=cuda).clone()
    v_d = torch.as_tensor(v0h, device=cuda).clone()
    pd = nat.ProjDesc(B, 3, tr.tiles_x, tr.tiles_y, tr.model_id, tr.max_group, 0, nat.ptr(pre))
    ad = nat.AdamDesc()
    for k in range(60):
        ad.lr[k] = float(lr[k])
    ad.beta1, ad.beta2, ad.eps, ad.step, ad.selective = B1, B2, EPS, step, selective
    nat.call("bs_project_bwd_adam", pd, ad, nat.ptr(p_d), nat.ptr(m_d), nat.ptr(v_d), tr.S, nat.ptr(mask),
             nat.ptr(tr.group_begin), tr.n_groups, nat.ptr(base), nat.ptr(v0), nat.ptr(cams), nat.ptr(gsp),
             nat.stream_handle())
    p_gpu, m_gpu, v_gpu = (t.cpu().numpy() for t in (p_d, m_d, v_d))
    # oracle Adam (dense), then restore the invisible points for selective Adam
    p_ref, m_ref, v_ref = params.copy(), m0.copy(), v0h.copy()
    py_oracle.adam(p_ref, g_ref, m_ref, v_ref, lr, B1, B2, EPS, step)
    vis = m_host != 0
    if selective:
        for a, b in ((p_ref, params), (m_ref, m0), (v_ref, v0h)):
            a[:, ~vis, :] = b[:, ~vis, :]
        assert np.array_equal(p_gpu[:, ~vis, :], params[:, ~vis, :])
        assert np.array_equal(m_gpu[:, ~vis, :], m0[:, ~vis, :])
    assert vis.any() and (~vis).any()
    # the gradient the kernel used, recovered from m' = m + (1 - b1)(g - m)
    # (selective Adam: over the visible points, the only ones it updates)
    g_used = (m_gpu.astype(np.float64) - B1 * m0.astype(np.float64)) / (1.0 - B1)
    upd = vis if selective else np.ones_like(vis)
    err = np.abs(g_used - g_ref)[:, upd, :].max(axis=1) / scale[:, 0, :]
    assert (err <= GRAD_REL).all(), err.max()
    # second moments and parameters against the oracle's Adam
    np.testing.assert_allclose(v_gpu, v_ref, rtol=1e-4, atol=1e-6 * float(scale.max()) ** 2)
    lr_full = np.broadcast_to(lr.reshape(15, 1, 4), params.shape)
    ulp = np.spacing(np.abs(p_ref).astype(np.float32))
    diff = np.abs(p_gpu - p_ref)
    assert (diff <= 2e-3 * lr_full + 4 * ulp).all(), (diff / (lr_full + 1e-30)).max()
    # and the parameters really moved by gradient-dependent amounts
    assert np.abs(p_gpu - params)[:, vis, :].max() > 0


def test_gsp_cleared_by_projection_over_three_steps(cuda):
    """Single-rank steps clear the G_SP accumulator inside the projection
    (bs_proj_desc.gsp_zero); the radix pipeline clears it with an explicit
    zero_().  Three training steps of both give the same parameters (a stale
    accumulator from step 1 would double-count step 2's gradient)."""
    ds, params, gb, aabb, gt = c1_setup()
    lr = scenes.lr_table(50.0)
    out = []
    for mode in ("bucket", "radix"):
        tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, sh_degree=3, adam=AdamConfig(lr))
        tr.binning = mode
        for b in ([0, 2, 5], [1, 3, 6], [0, 2, 5]):
            tr.step(b)
        torch.cuda.synchronize()
        out.append((tr.params.cpu().numpy(), tr.exp_avg.cpu().numpy()))
    (pa, ma), (pb, mb) = out
    lr_full = np.broadcast_to(lr.reshape(15, 1, 4), pa.shape)
    assert (np.abs(pa - pb) <= 1e-3 * lr_full + 4 * np.spacing(np.abs(pa))).all()
    mscale = np.abs(mb).reshape(15, -1, 4).max(axis=1, keepdims=True) + 1e-30
    assert (np.abs(ma - mb) / mscale).max() <= 1e-3


def test_checkpoint_resume(cuda, tmp_path):
    """state_dict / load_state_dict: resuming a saved shard (parameters, Adam
    moments, step counter) continues training exactly like the uninterrupted
    run (same kernels, same inputs; tolerance for atomic order only)."""
    ds, params, gb, aabb, gt = c1_setup()
    lr = scenes.lr_table(50.0)
    a = SplatTrainer(params, gb, aabb, ds.views, gt=gt, adam=AdamConfig(lr))
    a.step([0, 2, 5])
    a.step([1, 3, 6])
    torch.save(a.state_dict(), tmp_path / "ckpt.pt")
    b = SplatTrainer(params, gb, aabb, ds.views, gt=gt, adam=AdamConfig(lr))
    b.load_state_dict(torch.load(tmp_path / "ckpt.pt"))
    assert b.step_count == 2
    a.step([0, 4, 7])
    b.step([0, 4, 7])
    torch.cuda.synchronize()
    pa, pb = a.params.cpu().numpy(), b.params.cpu().numpy()
    lr_full = np.broadcast_to(lr.reshape(15, 1, 4), pa.shape)
    assert (np.abs(pa - pb) <= 1e-3 * lr_full + 4 * np.spacing(np.abs(pa))).all()
    from paper_2512_20017_b200.status import ConsistencyError

    c = SplatTrainer(params[:, :100], np.array([0, 100], dtype=np.int32), aabb[:1], ds.views, gt=gt)
    with pytest.raises(ConsistencyError):
        c.load_state_dict(a.state_dict())
