"""2DGS (surfel) half of the oracle (config 3, SURVEY.md §8 row "2D"),
pinned against an independent float64 torch-autograd restatement of the
surfel projection + ray-splat intersection + blending.  No GPU needed.

The paper's 2DGS kernels (gsplat) are absent from /root/reference, so this
half is "parity unpinned" against the reference itself;
the restatement below fixes the conventions of PAPER.md:1217-1226: 3x3 ray
transform M = [K Rcw t_u s_u, K Rcw t_v s_v, K Rcw (p - c)], intersection
(u, v) = (h_x x h_y).xy / (h_x x h_y).z, low-pass min(u^2 + v^2, 2 |d|^2)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import py_oracle
from paper_2512_20017_b200.trainer import camera_bytes
from _scene import c1_setup, oracle_view_pipeline
from test_oracle_cpu import SH_C0, SH_C1, SH_C2, SH_C3


def _t_project2d(mean, ls, quat, opl, sh, view):
    R = torch.as_tensor(view.rotation.T, dtype=torch.float64)  # world -> camera
    cpos = torch.as_tensor(np.float32(view.position).astype(np.float64))
    fx, fy, cx, cy = view.intrinsics()
    K = torch.tensor([[fx, 0.0, cx], [0.0, fy, cy], [0.0, 0.0, 1.0]], dtype=torch.float64)
    d = mean - cpos
    s = torch.exp(ls[:, :2])
    qn = quat / quat.norm(dim=1, keepdim=True)
    w, x, y, z = qn.unbind(1)
    Rq = torch.stack([
        1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
        2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
        2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1).view(-1, 3, 3)
    Rc = R @ Rq
    c0 = (Rc[:, :, 0] * s[:, :1]) @ K.T
    c1 = (Rc[:, :, 1] * s[:, 1:]) @ K.T
    c2 = (d @ R.T) @ K.T
    M = torch.stack([c0, c1, c2], 2)  # rows of M: (c0_i, c1_i, c2_i)
    u, v = c2[:, 0] / c2[:, 2], c2[:, 1] / c2[:, 2]
    dirv = d / d.norm(dim=1, keepdim=True)
    X, Y, Z = dirv.unbind(1)
    xx, yy, zz = X * X, Y * Y, Z * Z
    basis = [torch.full_like(X, SH_C0), -SH_C1 * Y, SH_C1 * Z, -SH_C1 * X,
             SH_C2[0] * X * Y, SH_C2[1] * Y * Z, SH_C2[2] * (2 * zz - xx - yy), SH_C2[3] * X * Z,
             SH_C2[4] * (xx - yy),
             SH_C3[0] * Y * (3 * xx - yy), SH_C3[1] * X * Y * Z, SH_C3[2] * Y * (4 * zz - xx - yy),
             SH_C3[3] * Z * (2 * zz - 3 * xx - 3 * yy), SH_C3[4] * X * (4 * zz - xx - yy),
             SH_C3[5] * Z * (xx - yy), SH_C3[6] * X * (xx - 3 * yy)]
    Yb = torch.stack(basis, 1)
    col = (torch.einsum("sk,skc->sc", Yb, sh.view(-1, 16, 3)) + 0.5).clamp(min=0)
    return u, v, M, col, torch.sigmoid(opl)


def _setup():
    ds, params, gb, aabb, gt = c1_setup(n_points=300, image_size=(48, 32), n_views=2, grid=(1, 1), G=64)
    view = ds.views[0]
    ref = oracle_view_pipeline(params, gb, aabb, view, camera_bytes([view]), gt[0], model="2dgs")
    return ds, params, gb, aabb, gt, view, ref


def test_project2d_rows_consistent_with_float64():
    """SP2 rows (mean2d, M, colour, depth, radii, normal) agree with the f64
    restatement; radii bound the 3-sigma disk image."""
    ds, params, gb, aabb, gt, view, ref = _setup()
    idx, sp = ref["idx"], ref["sp"]
    assert sp.shape == (len(idx), 24) and len(idx) > 50
    P = torch.as_tensor(params.astype(np.float64))
    sh = P[3:15, idx, :].permute(1, 0, 2).reshape(len(idx), 48)
    u, v, M, col, opac = _t_project2d(P[0, idx, :3], P[1, idx, :3], P[2, idx, :], P[0, idx, 3], sh, view)
    valid = sp[:, 16] > 0
    assert valid.mean() > 0.5
    np.testing.assert_allclose(sp[:, 0], u.numpy(), rtol=1e-4, atol=1e-3)
    np.testing.assert_allclose(sp[:, 1], v.numpy(), rtol=1e-4, atol=1e-3)
    np.testing.assert_allclose(sp[:, 3:12], M.reshape(-1, 9).numpy(), rtol=1e-4, atol=1e-3)
    np.testing.assert_allclose(sp[:, 12:15], col.numpy(), atol=1e-5)
    np.testing.assert_allclose(sp[:, 2], opac.numpy(), atol=1e-6)
    # the support box (centre sp[22:24], half-widths sp[16:18]) holds the disk
    # u^2 + v^2 <= k and the low-pass circle of radius sqrt(k / 2),
    # k = min(9, 2 ln(255 o))
    th = np.linspace(0, 2 * np.pi, 64, endpoint=False)
    Mn = M.numpy()
    for k in np.flatnonzero(valid)[:40]:
        kk = min(9.0, 2.0 * np.log(255.0 * float(sp[k, 2])))
        rk = np.sqrt(kk)
        pts = Mn[k] @ np.stack([rk * np.cos(th), rk * np.sin(th), np.ones_like(th)])
        px, py = pts[0] / pts[2], pts[1] / pts[2]
        px = np.concatenate([px, sp[k, 0] + np.sqrt(kk / 2) * np.cos(th)])
        py = np.concatenate([py, sp[k, 1] + np.sqrt(kk / 2) * np.sin(th)])
        assert np.all(np.abs(px - sp[k, 22]) <= sp[k, 16] * (1 + 1e-4) + 1e-3)
        assert np.all(np.abs(py - sp[k, 23]) <= sp[k, 17] * (1 + 1e-4) + 1e-3)
    # normal: unit, camera-facing
    n = sp[valid, 18:21]
    np.testing.assert_allclose(np.linalg.norm(n, axis=1), 1.0, atol=1e-5)


def test_oracle2d_gradients_match_float64_autograd():
    ds, params, gb, aabb, gt, view, ref = _setup()
    idx = ref["idx"]
    P = torch.as_tensor(params.astype(np.float64))
    mean = P[0, idx, :3].clone().requires_grad_(True)
    opl = P[0, idx, 3].clone().requires_grad_(True)
    ls = P[1, idx, :3].clone().requires_grad_(True)
    quat = P[2, idx, :].clone().requires_grad_(True)
    sh = P[3:15, idx, :].permute(1, 0, 2).reshape(len(idx), 48).clone().requires_grad_(True)
    u, v, M, col, opac = _t_project2d(mean, ls, quat, opl, sh, view)
    W, H = view.width, view.height
    tx = (W + 15) // 16
    img = []
    n_branch = [0, 0]
    for py in range(H):
        for px in range(W):
            t = (py // 16) * tx + px // 16
            r0, _ = ref["ranges"][t]
            cand = ref["lists"][r0:r0 + ref["nc"][py, px]].astype(np.int64)
            if len(cand) == 0:
                img.append(torch.zeros(3, dtype=torch.float64))
                continue
            ci = torch.as_tensor(cand)
            x, y = px + 0.5, py + 0.5
            Mc = M[ci]
            hx = Mc[:, 0, :] - x * Mc[:, 2, :]
            hy = Mc[:, 1, :] - y * Mc[:, 2, :]
            zeta = torch.cross(hx, hy, dim=1)
            uu, vv = zeta[:, 0] / zeta[:, 2], zeta[:, 1] / zeta[:, 2]
            g3 = uu * uu + vv * vv
            g2 = 2 * ((u[ci] - x) ** 2 + (v[ci] - y) ** 2)
            use3 = (g3 <= g2).detach()
            n_branch[0] += int(use3.sum())
            n_branch[1] += int((~use3).sum())
            power = -0.5 * torch.where(use3, g3, g2)
            alpha = (opac[ci] * torch.exp(power)).clamp(max=0.99)
            keep = (power.detach() <= 0) & (power.detach() >= -4.5) & (alpha.detach() >= 1.0 / 255.0)
            alpha = alpha[keep]
            cc = col[ci][keep]
            T = torch.cumprod(torch.cat([torch.ones(1, dtype=torch.float64), 1 - alpha[:-1]]), 0)
            img.append((cc * (alpha * T)[:, None]).sum(0))
    assert min(n_branch) > 0, n_branch  # both the surfel and the low-pass branch are exercised
    img = torch.stack(img).view(H, W, 3)
    np.testing.assert_allclose(img.detach().numpy(), ref["img"], atol=5e-5)
    loss = (img - torch.as_tensor(gt[0].astype(np.float64) / 255.0)).abs().mean()
    loss.backward()
    g = ref["gparams"]
    checks = {
        "mean": (mean.grad.numpy(), g[0, idx, :3]),
        "opacity": (opl.grad.numpy(), g[0, idx, 3]),
        "log_scale": (ls.grad.numpy()[:, :2], g[1, idx, :2]),
        "quat": (quat.grad.numpy(), g[2, idx, :]),
        "sh": (sh.grad.numpy(), g[3:15, idx, :].transpose(1, 0, 2).reshape(len(idx), 48)),
    }
    for name, (auto, mine) in checks.items():
        scale = np.abs(auto).max()
        assert scale > 0, name
        err = np.abs(auto - mine).max() / scale
        assert err < 2e-3, (name, err)
    assert np.all(g[1, idx, 2] == 0)  # the third scale is unused by surfels


def test_oracle2d_train_step_runs_and_decreases_loss():
    ds, params, gb, aabb, gt, view, ref = _setup()
    from paper_2512_20017_b200.culling import batch_planes

    p = params.copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    lr = np.full(60, 1e-3, dtype=np.float32)
    cams = camera_bytes(ds.views[:1])
    planes = batch_planes(ds.views[:1], 1)
    losses = [py_oracle.train_step(p, m, v, planes, cams, gt[:1], 3, lr, 0.9, 0.999, 1e-15, s + 1, model="2dgs")
              for s in range(4)]
    assert np.all(np.isfinite(losses))
    assert losses[-1] < losses[0]
