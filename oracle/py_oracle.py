"""ctypes wrapper of oracle/splat_oracle.c (TEST INFRASTRUCTURE ONLY).

numpy in, numpy out.  See splat_oracle.h for what each function restates and
which reference file:line it follows.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "build", "libsplat_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "splat_oracle.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_LIB), exist_ok=True)
        subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC",
                        "-shared", "-o", _LIB, src, "-lm"], check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        P, I32, I64, F, D = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_double
        sig = {
            "or_access_matrix": (None, [P, I64, P, P, I32, P, I32, I32, P, I32, I32, P, P, P]),
            "or_visibility_mask": (None, [P, I64, P, P, I32, P, I32, P]),
            "or_morton": (None, [P, I64, P, I32, P]),
            "or_det_expf": (F, [F]),
            "or_det_logf": (F, [F]),
            "or_project": (None, [P, I64, P, I64, P, I32, P]),
            "or_project_bwd": (None, [P, I64, P, I64, P, I32, P, P]),
            "or_render": (I32, [P, I64, I32, I32, P, P, P, P, P, P, P]),
            "or_render_bwd": (I32, [P, I64, I32, I32, P, P, P, P, P]),
            "or_l1_loss": (D, [P, P, I64, P]),
            "or_adam": (None, [P, P, P, P, I64, P, I64, F, F, F, I32]),
            "or_train_step": (D, [P, P, P, I64, P, P, I32, P, I32, P, F, F, F, I32, I32]),
            "or_plane_distances": (None, [P, I64, P, I32, P]),
            "or_project2d": (None, [P, I64, P, I64, P, I32, P]),
            "or_project2d_bwd": (None, [P, I64, P, I64, P, I32, P, P]),
            "or_render2d": (I32, [P, I64, I32, I32, P, P, P, P, P, P, P]),
            "or_render2d_bwd": (I32, [P, I64, I32, I32, P, P, P, P, P]),
            "or_train_step_model": (D, [P, P, P, I64, P, P, I32, P, I32, P, F, F, F, I32, I32, I32]),
            "so_densify_mark": (None, [P, I64, P, P, I32, F, F, F, F, P, P]),
            "so_densify_apply": (None, [P, P, P, I64, P, P, P, I32, P, C.c_uint32, P, P, P, I64, P]),
            "so_group_aabb_ranges": (None, [P, P, I32, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def access_matrix(positions, group_begin, aabb, planes, B, P, point_gpu, N, mode=0, presence=None,
                  view_times=None):
    pos = _c(positions, np.float32)
    gb = _c(group_begin, np.int32)
    ab = None if aabb is None else _c(aabb, np.float32)
    pl = _c(planes, np.float64)
    pg = None if point_gpu is None else _c(point_gpu, np.int32)
    pr = None if presence is None else _c(presence, np.float32)
    vt = None if view_times is None else _c(view_times, np.float32)
    out = np.zeros((B * P * P, N), dtype=np.int64)
    lib().or_access_matrix(_p(pos), len(pos), _p(gb), _p(ab), len(gb) - 1, _p(pl), B, P, _p(pg), N, mode, _p(pr),
                           _p(vt), _p(out))
    return out


def visibility_mask(positions, group_begin, aabb, planes, B):
    pos = _c(positions, np.float32)
    gb = _c(group_begin, np.int32)
    ab = None if aabb is None else _c(aabb, np.float32)
    pl = _c(planes, np.float64)
    out = np.zeros(len(pos), dtype=np.uint32)
    lib().or_visibility_mask(_p(pos), len(pos), _p(gb), _p(ab), len(gb) - 1, _p(pl), B, _p(out))
    return out


def plane_distances(points, planes):
    """fma(z, c, fma(y, b, x*a)) + d for every (point, plane) -- the kernels' order."""
    pts = _c(points, np.float64)
    pl = _c(planes, np.float64)
    out = np.zeros((len(pts), len(pl)), dtype=np.float64)
    lib().or_plane_distances(_p(pts), len(pts), _p(pl), len(pl), _p(out))
    return out


def morton(positions, bbox, bits):
    pos = _c(positions, np.float32)
    bb = _c(bbox, np.float32).reshape(6)
    out = np.zeros(len(pos), dtype=np.uint64)
    lib().or_morton(_p(pos), len(pos), _p(bb), bits, _p(out))
    return out


def det_expf(x: float) -> float:
    return lib().or_det_expf(float(x))


def det_logf(x: float) -> float:
    return lib().or_det_logf(float(x))


# row widths per model: 3DGS SP 12 / G_SP 9, 2DGS SP 24 / G_SP 15 (include/splat_b200.h)
_WIDTH = {"3dgs": (12, 9, ""), "2dgs": (24, 15, "2d")}


def project(params, idx, cam_bytes, sh_degree, model="3dgs"):
    spf, _, sfx = _WIDTH[model]
    prm = _c(params, np.float32)
    S = prm.shape[1]
    ix = _c(idx, np.int64)
    cam = _c(cam_bytes, np.uint8)
    out = np.zeros((len(ix), spf), dtype=np.float32)
    getattr(lib(), "or_project" + sfx)(_p(prm), S, _p(ix), len(ix), _p(cam), sh_degree, _p(out))
    return out


def project_bwd(params, idx, cam_bytes, sh_degree, gsp, grad=None, model="3dgs"):
    _, _, sfx = _WIDTH[model]
    prm = _c(params, np.float32)
    S = prm.shape[1]
    ix = _c(idx, np.int64)
    cam = _c(cam_bytes, np.uint8)
    g = _c(gsp, np.float32)
    out = np.zeros_like(prm) if grad is None else grad
    getattr(lib(), "or_project" + sfx + "_bwd")(_p(prm), S, _p(ix), len(ix), _p(cam), sh_degree, _p(g), _p(out))
    return out


def render(sp, W, H, bg=(0.0, 0.0, 0.0), want_lists=False, model="3dgs"):
    _, _, sfx = _WIDTH[model]
    fn = getattr(lib(), "or_render" + sfx)
    s = _c(sp, np.float32)
    bgv = _c(bg, np.float32)
    img = np.zeros((H, W, 3), dtype=np.float32)
    T = np.zeros((H, W), dtype=np.float32)
    nc = np.zeros((H, W), dtype=np.int32)
    tx, ty = (W + 15) // 16, (H + 15) // 16
    if not want_lists:
        fn(_p(s), len(s), W, H, _p(bgv), _p(img), _p(T), _p(nc), None, None, None)
        return img, T, nc
    n = C.c_int64(0)
    ranges = np.zeros((tx * ty, 2), dtype=np.int32)
    fn(_p(s), len(s), W, H, _p(bgv), _p(img), _p(T), _p(nc), None, C.byref(n), None)
    lists = np.zeros(max(n.value, 1), dtype=np.uint32)
    rc = fn(_p(s), len(s), W, H, _p(bgv), _p(img), _p(T), _p(nc), _p(lists), C.byref(n), _p(ranges))
    assert rc == 0
    return img, T, nc, lists[: n.value], ranges


def render_bwd(sp, W, H, final_T, n_contrib, grad_image, bg=(0.0, 0.0, 0.0), model="3dgs"):
    _, gspf, sfx = _WIDTH[model]
    s = _c(sp, np.float32)
    bgv = _c(bg, np.float32)
    out = np.zeros((len(s), gspf), dtype=np.float32)
    getattr(lib(), "or_render" + sfx + "_bwd")(_p(s), len(s), W, H, _p(bgv), _p(_c(final_T, np.float32)),
                                               _p(_c(n_contrib, np.int32)), _p(_c(grad_image, np.float32)),
                                               _p(out))
    return out


def l1_loss(image, gt):
    img = _c(image, np.float32)
    g = _c(gt, np.uint8)
    grad = np.zeros_like(img)
    loss = lib().or_l1_loss(_p(img), _p(g), img.size, _p(grad))
    return loss, grad


def adam(params, grads, m, v, lr60, beta1, beta2, eps, step):
    S = params.shape[1]
    lib().or_adam(_p(params), _p(_c(grads, np.float32)), _p(m), _p(v), params.size, _p(_c(lr60, np.float32)), S,
                  beta1, beta2, eps, step)


def train_step(params, m, v, planes, cam_bytes, gt, sh_degree, lr60, beta1, beta2, eps, step, threads=0,
               model="3dgs"):
    """In-place CPU training step over len(cam_bytes) views; returns summed loss."""
    S = params.shape[1]
    B = len(cam_bytes)
    return lib().or_train_step_model(_p(params), _p(m), _p(v), S, _p(_c(planes, np.float64)),
                                     _p(_c(cam_bytes, np.uint8)), B, _p(_c(gt, np.uint8)), sh_degree,
                                     _p(_c(lr60, np.float32)), beta1, beta2, eps, step, threads,
                                     1 if model == "2dgs" else 0)


def zorder_layout(positions, G):
    """Host restatement of zorder_group (visibility.py:113-134): stable argsort
    of the oracle Morton codes, groups of G with float32 AABBs.
    Returns (perm int64, group_begin int32 [ng+1], aabb float32 [ng, 6])."""
    pos = np.ascontiguousarray(positions, dtype=np.float32)
    bbox = np.stack([pos.min(0), pos.max(0)])
    perm = np.argsort(morton(pos, bbox, 21), kind="stable")
    spos = pos[perm]
    n = len(pos)
    gb = np.concatenate([np.arange(0, n, G), [n]]).astype(np.int32)
    aabb = np.stack([np.concatenate([spos[b:e].min(0), spos[b:e].max(0)]) for b, e in zip(gb[:-1], gb[1:])])
    return perm, gb, aabb.astype(np.float32)


def densify(params, m, v, stats, group_begin, grad_threshold, split_scale, min_opacity, max_scale=0.0, seed=0,
            gid=None):
    """Clone / split / prune of a 3DGS shard (csrc/densify.cu semantics).
    params, m, v: float32 [15, S, 4]; stats float32 [S, 2] or None.
    Returns (action, group_out, new_group_begin, params', m', v', src_index, aabb')."""
    L = lib()
    params, m, v = (_c(a, np.float32) for a in (params, m, v))
    S = params.shape[1]
    gb = _c(group_begin, np.int32)
    ng = len(gb) - 1
    st = None if stats is None else _c(stats, np.float32)
    action = np.zeros(S, np.int32)
    gout = np.zeros(ng, np.int32)
    L.so_densify_mark(params.ctypes.data, S, _p(st), gb.ctypes.data, ng, grad_threshold, split_scale, min_opacity,
                      max_scale, action.ctypes.data, gout.ctypes.data)
    nb = np.zeros(ng + 1, np.int32)
    nb[1:] = np.cumsum(gout)
    Sn = int(nb[-1])
    pn = np.zeros((15, Sn, 4), np.float32)
    mn = np.zeros_like(pn)
    vn = np.zeros_like(pn)
    src = np.zeros(Sn, np.int32)
    g = None if gid is None else _c(gid, np.int32)
    L.so_densify_apply(params.ctypes.data, m.ctypes.data, v.ctypes.data, S, action.ctypes.data, gb.ctypes.data,
                       nb.ctypes.data, ng, _p(g), int(seed) & 0xFFFFFFFF, pn.ctypes.data, mn.ctypes.data,
                       vn.ctypes.data, Sn, src.ctypes.data)
    aabb = np.zeros((ng, 6), np.float32)
    L.so_group_aabb_ranges(pn.ctypes.data, nb.ctypes.data, ng, aabb.ctypes.data)
    return action, gout, nb, pn, mn, vn, src, aabb
