"""CPU tests: the oracle against the reference's golden vectors, the host data
model against the reference generators, and the oracle's analytic backward
against an independent float64 torch-autograd restatement.  No GPU needed."""

import math

import numpy as np
import pytest
import torch

from oracle import py_oracle
from paper_2512_20017_b200 import scenes
from paper_2512_20017_b200.culling import Frustum, batch_planes, cull_group, frustum_from_view, patch_frusta
from paper_2512_20017_b200.trainer import camera_bytes

from _scene import c1_setup, oracle_view_pipeline


def _aerial():
    return scenes.generate_aerial_scene(seed=3, n_points=6000, grid=(2, 3), n_views=10, altitude=20,
                                        image_size=(96, 64))


def _street():
    wps = [(0, 0, 0), (60, 0, 0), (60, 50, 0), (120, 50, 0)]
    return scenes.generate_street_scene(seed=4, n_points=3000, trajectory_waypoints=wps, n_views=12,
                                        image_size=(80, 60), duration=5.0)


# ---------------------------------------------------------------- data model


def test_generators_bit_identical_to_reference(golden):
    ds = _aerial()
    assert np.array_equal(ds.cloud.positions, golden["aerial_positions"])
    assert np.array_equal(np.stack([v.position for v in ds.views]), golden["aerial_cam_pos"])
    assert np.array_equal(np.stack([v.rotation for v in ds.views]), golden["aerial_cam_rot"])
    st = _street()
    assert np.array_equal(st.cloud.positions, golden["street_positions"])
    assert np.array_equal(st.cloud.timestamps, golden["street_presence"])
    assert np.array_equal(np.stack([v.position for v in st.views]), golden["street_cam_pos"])
    assert np.array_equal(np.stack([v.rotation for v in st.views]), golden["street_cam_rot"])
    assert np.array_equal(np.array([v.far for v in st.views]), golden["street_cam_far"])
    assert np.array_equal(np.array([v.time for v in st.views]), golden["street_view_times"])


@pytest.mark.parametrize("P", [1, 2, 3])
def test_frusta_planes_bit_identical(golden, P):
    fr = np.stack([f.planes for f in patch_frusta(_aerial().views[4], P)])
    assert np.array_equal(fr, golden[f"frusta_P{P}"])


def test_shared_plane_block_reproduces_patch_frusta():
    ds = _aerial()
    for P in (1, 2, 4):
        block = batch_planes([ds.views[2]], P)[0]
        for r in range(P):
            for c in range(P):
                f = patch_frusta(ds.views[2], P)[r * P + c]
                assert np.array_equal(f.planes[0], block[0]) and np.array_equal(f.planes[1], block[1])
                assert np.array_equal(f.planes[2], block[2 + c])
                assert np.array_equal(f.planes[3], -block[2 + c + 1])
                assert np.array_equal(f.planes[4], block[3 + P + r])
                assert np.array_equal(f.planes[5], -block[3 + P + r + 1])


def test_blas_distance_order_matches_plane_kernel_formula():
    """The kernels evaluate fma(z, c, fma(y, b, x*a)) + d; check it against
    the numpy/BLAS expression the reference uses (visibility.py:155-156)."""
    rng = np.random.default_rng(0)
    ds = _aerial()
    fr = frustum_from_view(ds.views[3])
    for n in (2, 3, 8, 17, 1000, 20000):
        pts = rng.uniform(-20, 80, (n, 3)).astype(np.float32).astype(np.float64)
        assert np.array_equal(py_oracle.plane_distances(pts, fr.planes), fr.signed_distances(pts)), n


def test_host_cull_api_shapes():
    ds = _aerial()
    fr = frustum_from_view(ds.views[0])
    assert isinstance(fr, Frustum) and fr.planes.shape == (6, 4)
    assert cull_group(fr, np.array([[1e6, 1e6, 1e6], [1e6 + 1, 1e6 + 1, 1e6 + 1]])) == "outside"


# ---------------------------------------------------------------- oracle integer half vs reference


def test_oracle_morton_matches_reference(golden):
    for bits in (1, 4, 10, 21):
        assert np.array_equal(py_oracle.morton(golden["morton_pts"], golden["morton_bbox"], bits),
                              golden[f"morton_codes_b{bits}"])
    flat = golden["morton_flat_pts"]
    assert np.array_equal(py_oracle.morton(flat, np.stack([flat.min(0), flat.max(0)]), 21),
                          golden["morton_flat_codes"])


def test_oracle_zorder_matches_reference(golden):
    perm, gb, aabb = py_oracle.zorder_layout(_aerial().cloud.positions, 128)
    assert np.array_equal(perm, golden["aerial_perm"])
    assert np.array_equal(aabb.reshape(-1, 2, 3), golden["aerial_aabb"])


@pytest.mark.parametrize("P", [1, 2, 3])
def test_oracle_access_matrix_matches_reference(golden, P):
    ds = _aerial()
    perm, gb, aabb = py_oracle.zorder_layout(ds.cloud.positions, 128)
    spos = ds.cloud.positions[perm]
    pl = batch_planes(ds.views, P)
    for mode, key in ((0, "exact"), (1, "group")):
        A = py_oracle.access_matrix(spos, gb, aabb, pl, len(ds.views), P, golden["aerial_point_gpu"], 3, mode)
        assert np.array_equal(A, golden[f"access_{key}_P{P}"])


def test_oracle_temporal_access_matches_reference(golden):
    st = _street()
    perm, gb, aabb = py_oracle.zorder_layout(st.cloud.positions, 64)
    assert np.array_equal(perm, golden["street_perm"])
    t = np.array([v.time for v in st.views], dtype=np.float32)
    A = py_oracle.access_matrix(st.cloud.positions[perm], gb, aabb, batch_planes(st.views, 2), 12, 2,
                                golden["street_point_gpu"], 2, 0, st.cloud.timestamps[perm], t)
    assert np.array_equal(A, golden["street_access_temporal_P2"])


def test_oracle_visibility_mask_matches_reference(golden):
    ds = _aerial()
    perm, gb, aabb = py_oracle.zorder_layout(ds.cloud.positions, 128)
    m = py_oracle.visibility_mask(ds.cloud.positions[perm], gb, aabb, batch_planes(ds.views, 1), 10)
    assert np.array_equal(m, golden["aerial_vis_mask"])


def test_det_expf_accuracy():
    xs = np.linspace(-30, 10, 2001, dtype=np.float32)
    got = np.array([py_oracle.det_expf(x) for x in xs], dtype=np.float64)
    ref = np.exp(xs.astype(np.float64))
    assert (np.abs(got - ref) / ref).max() < 5e-7


def test_det_logf_accuracy():
    """Deterministic ln used for the opacity-aware support extents
    k = min(9, 2 ln(255 o)) (csrc/common.cuh det_logf)."""
    xs = np.concatenate([np.geomspace(1e-30, 1e30, 3001), np.linspace(0.5, 2.0, 2001),
                         255.0 * np.linspace(1e-4, 1.0, 2001)]).astype(np.float32)
    got = np.array([py_oracle.det_logf(x) for x in xs], dtype=np.float64)
    ref = np.log(xs.astype(np.float64))
    err = np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)
    assert err.max() < 3e-7
    assert py_oracle.det_logf(0.0) == -87.5 and py_oracle.det_logf(-1.0) == -87.5


# ---------------------------------------------------------------- float half: oracle vs f64 autograd


SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = [1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792, 0.5462742152960396]
SH_C3 = [-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154, -0.4570457994644658,
         1.445305721320277, -0.5900435899266435]


def _t_project(mean, ls, quat, opl, sh, view):
    """float64 torch restatement of pts_splatting (splat_math.cuh conventions)."""
    R = torch.as_tensor(view.rotation.T, dtype=torch.float64)
    cpos = torch.as_tensor(np.float32(view.position).astype(np.float64))
    fx, fy, cx, cy = view.intrinsics()
    limx, limy = 1.3 * math.tan(view.fov_x / 2), 1.3 * math.tan(view.fov_y / 2)
    d = mean - cpos
    q = d @ R.T
    z = q[:, 2]
    s = torch.exp(ls)
    qn = quat / quat.norm(dim=1, keepdim=True)
    w, x, y, zq = qn.unbind(1)
    Rq = torch.stack([
        1 - 2 * (y * y + zq * zq), 2 * (x * y - w * zq), 2 * (x * zq + w * y),
        2 * (x * y + w * zq), 1 - 2 * (x * x + zq * zq), 2 * (y * zq - w * x),
        2 * (x * zq - w * y), 2 * (y * zq + w * x), 1 - 2 * (x * x + y * y)], 1).view(-1, 3, 3)
    M = Rq * s[:, None, :]
    Sg = M @ M.transpose(1, 2)
    Sc = R @ Sg @ R.T
    xr, yr = q[:, 0] / z, q[:, 1] / z
    tx = xr.clamp(-limx, limx) * z
    ty = yr.clamp(-limy, limy) * z
    zero = torch.zeros_like(z)
    J = torch.stack([torch.stack([fx / z, zero, -fx * tx / z ** 2], 1),
                     torch.stack([zero, fy / z, -fy * ty / z ** 2], 1)], 1)
    cov = J @ Sc @ J.transpose(1, 2)
    a, b, c = cov[:, 0, 0] + 0.3, cov[:, 0, 1], cov[:, 1, 1] + 0.3
    det = a * c - b * b
    conic = torch.stack([c / det, -b / det, a / det], 1)
    u, v = fx * xr + cx, fy * yr + cy
    dirv = d / d.norm(dim=1, keepdim=True)
    X, Y, Z = dirv.unbind(1)
    xx, yy, zz = X * X, Y * Y, Z * Z
    basis = [torch.full_like(X, SH_C0), -SH_C1 * Y, SH_C1 * Z, -SH_C1 * X,
             SH_C2[0] * X * Y, SH_C2[1] * Y * Z, SH_C2[2] * (2 * zz - xx - yy), SH_C2[3] * X * Z,
             SH_C2[4] * (xx - yy),
             SH_C3[0] * Y * (3 * xx - yy), SH_C3[1] * X * Y * Z, SH_C3[2] * Y * (4 * zz - xx - yy),
             SH_C3[3] * Z * (2 * zz - 3 * xx - 3 * yy), SH_C3[4] * X * (4 * zz - xx - yy),
             SH_C3[5] * Z * (xx - yy), SH_C3[6] * X * (xx - 3 * yy)]
    Yb = torch.stack(basis, 1)  # (S, 16)
    col = (torch.einsum("sk,skc->sc", Yb, sh.view(-1, 16, 3)) + 0.5).clamp(min=0)
    opac = torch.sigmoid(opl)
    return u, v, conic, col, opac


def test_oracle_gradients_match_float64_autograd():
    """Pins the hand-derived backward (oracle, same formulas as the kernels)
    against autograd of an independent float64 restatement: tiny scene."""
    ds, params, gb, aabb, gt = c1_setup(n_points=300, image_size=(48, 32), n_views=2, grid=(1, 1), G=64)
    view = ds.views[0]
    ref = oracle_view_pipeline(params, gb, aabb, view, camera_bytes([view]), gt[0])
    idx = ref["idx"]
    assert len(idx) > 50
    P = torch.as_tensor(params.astype(np.float64))
    mean = P[0, idx, :3].clone().requires_grad_(True)
    opl = P[0, idx, 3].clone().requires_grad_(True)
    ls = P[1, idx, :3].clone().requires_grad_(True)
    quat = P[2, idx, :].clone().requires_grad_(True)
    sh = P[3:15, idx, :].permute(1, 0, 2).reshape(len(idx), 48).clone().requires_grad_(True)
    u, v, conic, col, opac = _t_project(mean, ls, quat, opl, sh, view)
    # blend with the oracle's discrete decisions (tile lists, n_contrib)
    W, H = view.width, view.height
    tx = (W + 15) // 16
    img = []
    for py in range(H):
        for px in range(W):
            t = (py // 16) * tx + px // 16
            r0, _ = ref["ranges"][t]
            cand = ref["lists"][r0:r0 + ref["nc"][py, px]].astype(np.int64)
            if len(cand) == 0:
                img.append(torch.zeros(3, dtype=torch.float64))
                continue
            ci = torch.as_tensor(cand)
            dx, dy = u[ci] - (px + 0.5), v[ci] - (py + 0.5)
            A, Bc, Cc = conic[ci, 0], conic[ci, 1], conic[ci, 2]
            power = -0.5 * (A * dx * dx + Cc * dy * dy) - Bc * dx * dy
            alpha = (opac[ci] * torch.exp(power)).clamp(max=0.99)
            keep = (power.detach() <= 0) & (power.detach() >= -4.5) & (alpha.detach() >= 1.0 / 255.0)
            alpha = alpha[keep]
            cc = col[ci][keep]
            T = torch.cumprod(torch.cat([torch.ones(1, dtype=torch.float64), 1 - alpha[:-1]]), 0)
            img.append((cc * (alpha * T)[:, None]).sum(0))
    img = torch.stack(img).view(H, W, 3)
    np.testing.assert_allclose(img.detach().numpy(), ref["img"], atol=2e-5)
    loss = (img - torch.as_tensor(gt[0].astype(np.float64) / 255.0)).abs().mean()
    loss.backward()
    g = ref["gparams"]
    checks = {
        "mean": (mean.grad.numpy(), g[0, idx, :3]),
        "opacity": (opl.grad.numpy(), g[0, idx, 3]),
        "log_scale": (ls.grad.numpy(), g[1, idx, :3]),
        "quat": (quat.grad.numpy(), g[2, idx, :]),
        "sh": (sh.grad.numpy(), g[3:15, idx, :].transpose(1, 0, 2).reshape(len(idx), 48)),
    }
    for name, (auto, mine) in checks.items():
        scale = np.abs(auto).max()
        assert scale > 0, name
        err = np.abs(auto - mine).max() / scale
        assert err < 2e-3, (name, err)


def test_oracle_adam_matches_torch():
    rng = np.random.default_rng(2)
    S = 50
    p = rng.normal(0, 1, (15, S, 4)).astype(np.float32)
    lr = rng.uniform(1e-4, 1e-2, 60).astype(np.float32)
    m, v = np.zeros_like(p), np.zeros_like(p)
    ref = [torch.nn.Parameter(torch.as_tensor(p[k // 4, :, k % 4].copy())) for k in range(60)]
    opts = [torch.optim.Adam([t], lr=float(lr[k]), eps=1e-15) for k, t in enumerate(ref)]
    for step in range(1, 5):
        g = rng.normal(0, 1e-2, p.shape).astype(np.float32)
        py_oracle.adam(p, g, m, v, lr, 0.9, 0.999, 1e-15, step)
        for k, (t, o) in enumerate(zip(ref, opts)):
            t.grad = torch.as_tensor(g[k // 4, :, k % 4].copy())
            o.step()
    for k, t in enumerate(ref):
        np.testing.assert_allclose(p[k // 4, :, k % 4], t.detach().numpy(), rtol=1e-5, atol=1e-7)
