"""The paper's user-defined-function protocol (Fig. sys-api)
over the C ABI: `pts_culling`, `pts_splatting`, `image_render`, the last two
differentiable as torch.autograd.Functions.  The reference package has no
such API ("the paper UDF protocol that the reference lacks");
this is the per-view, single-GPU form of what trainer.SplatTrainer fuses
across a batch.

Point-cloud state PC is a dict of [S, l] tensors on the GPU:
  xyz [S, 3], opacity [S, 1] (logit), scaling [S, 3] (log; 2DGS uses x, y),
  rotation [S, 4] (w, x, y, z), sh [S, 16, 3] (degree-3 SH, coefficient-major)
  and, for temporal culling, presence [S, 2].
Splats SP are a dict of [V, l] tensors over the in-frustum points:
  3DGS: means2d [V, 2], opacities [V], conics [V, 3], colors [V, 3],
        depths [V], radii [V, 2]
  2DGS: means2d [V, 2], opacities [V], ray_transforms [V, 9] (KWH, row-major),
        colors [V, 3], depths [V], radii [V, 2], normals [V, 3]
                                         
Gradients flow to every float element except depths, radii and normals
(integer-like or unused by the L1 image loss).  There is no CPU path: every
call raises NativeError without the kernel library or a GPU.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as nat
from .binning import bin_buckets
from .culling import view_plane_block
from .scenes import CameraView

_CHUNK = 256  # points per CTA of the per-point kernels
_MODELS = {"3dgs": nat.MODEL_3DGS, "2dgs": nat.MODEL_2DGS}


class _Buffers:
    """Grow-only device buffers (per call site)."""

    def __init__(self):
        self.bufs = {}

    def get(self, name, n, dtype):
        b = self.bufs.get(name)
        if b is None or b.numel() < n or b.dtype != dtype:
            b = torch.empty(max(int(n * 1.25) + 1024, 1024), dtype=dtype, device=torch.cuda.current_device())
            self.bufs[name] = b
        return b[:n]


_buf = _Buffers()


def _camera(view: CameraView, dev) -> torch.Tensor:
    from .trainer import camera_bytes

    return torch.as_tensor(camera_bytes([view]), device=dev)


def _chunk_groups(n: int, dev):
    """Groups of _CHUNK consecutive points: (group_begin int32, n_groups)."""
    gb = np.minimum(np.arange(0, n + _CHUNK, _CHUNK), n)
    gb = np.unique(gb).astype(np.int32)
    return torch.as_tensor(gb, device=dev), len(gb) - 1


# ---------------------------------------------------------------- pts_culling


def pts_culling(view: CameraView, PC: dict, view_time: float | None = None) -> torch.Tensor:
    """Indices (int64, ascending) of the points of PC inside the view frustum
    (K0, visibility.py:153-161 semantics: near/far and edge planes in f64).
    With view_time, also requires presence[:, 0] <= t <= presence[:, 1] (f32)."""
    nat.load()
    xyz = PC["xyz"].detach().float().contiguous()
    dev, S = xyz.device, xyz.shape[0]
    if S == 0:
        return torch.empty(0, dtype=torch.int64, device=dev)
    gb, ng = _chunk_groups(S, dev)
    planes = torch.as_tensor(view_plane_block(view, 1)[None], device=dev)
    temporal = view_time is not None
    presence = times = None
    if temporal:
        if "presence" not in PC:
            from .status import ConfigurationError

            raise ConfigurationError("temporal culling needs PC['presence']")
        presence = PC["presence"].detach().float().contiguous()
        times = torch.tensor([view_time], dtype=torch.float32, device=dev)
    mask = torch.empty(S, dtype=torch.int32, device=dev)
    counts = torch.empty(ng, dtype=torch.int32, device=dev)
    desc = nat.CullDesc(nat.CULL_MASK, 1, 1, 1, 1 if temporal else 0, 3)
    nat.call("bs_cull_count", desc, nat.ptr(xyz), S, nat.ptr(presence), nat.ptr(gb), None, ng, nat.ptr(planes),
             nat.ptr(times), None, nat.ptr(mask), nat.ptr(counts), None, nat.stream_handle())
    return torch.nonzero(mask != 0).flatten()


# ---------------------------------------------------------------- pts_splatting


def pack_points(PC: dict, ids: torch.Tensor) -> torch.Tensor:
    """Differentiable gather of the in-frustum points into the kernels'
    plane-major layout [15, V, 4] (include/splat_b200.h)."""
    V = ids.numel()
    xyz = PC["xyz"][ids]
    opac = PC["opacity"].reshape(-1, 1)[ids]
    scl = PC["scaling"][ids]
    if scl.shape[1] == 2:
        scl = torch.cat([scl, torch.zeros_like(scl[:, :1])], 1)
    rot = PC["rotation"][ids]
    sh = PC["sh"].reshape(PC["sh"].shape[0], -1)[ids]
    if sh.shape[1] < 48:
        sh = torch.cat([sh, sh.new_zeros(V, 48 - sh.shape[1])], 1)
    p0 = torch.cat([xyz, opac], 1)
    p1 = torch.cat([scl, torch.zeros_like(scl[:, :1])], 1)
    planes = torch.stack([p0, p1, rot], 0)
    planes = torch.cat([planes, sh.reshape(V, 12, 4).permute(1, 0, 2)], 0)
    return planes.float().contiguous()


class _ProjectFn(torch.autograd.Function):
    """planes [15, V, 4] -> splat rows [V, SP] (K1) / grad rows -> grad planes (K1b)."""

    @staticmethod
    def forward(ctx, planes, cam, view_wh, sh_degree, model_id):
        V = planes.shape[1]
        dev = planes.device
        width = nat.SP2_FLOATS if model_id == nat.MODEL_2DGS else nat.SP_FLOATS
        sp = torch.empty((V, width), dtype=torch.float32, device=dev)
        ctx.model_id, ctx.sh_degree = model_id, sh_degree
        if V == 0:
            ctx.save_for_backward(planes, cam)
            return sp
        gb, ng = _chunk_groups(V, dev)
        mask = torch.ones(V, dtype=torch.int32, device=dev)  # every packed point is visible in view 0
        counts = (gb[1:] - gb[:-1]).to(torch.int32).contiguous()
        base = torch.empty(ng, dtype=torch.int32, device=dev)
        rows = torch.empty(1, dtype=torch.int64, device=dev)
        row0 = torch.empty(1, dtype=torch.int64, device=dev)
        st = nat.stream_handle()
        nat.call("bs_scan_counts", nat.ptr(counts), ng, 1, None, nat.ptr(base), nat.ptr(rows), nat.ptr(row0), st)
        tx, ty = (view_wh[0] + 15) // 16, (view_wh[1] + 15) // 16
        desc = nat.ProjDesc(1, sh_degree, tx, ty, model_id, _CHUNK)
        nat.call("bs_project_fwd", desc, nat.ptr(planes), V, nat.ptr(mask), nat.ptr(gb), ng, nat.ptr(base),
                 nat.ptr(row0), nat.ptr(cam), nat.ptr(sp), st)
        ctx.save_for_backward(planes, cam, mask, gb, base, row0)
        ctx.ng = ng
        return sp

    @staticmethod
    def backward(ctx, grad_sp):
        if grad_sp is None or ctx.saved_tensors[0].shape[1] == 0:
            return None, None, None, None, None
        planes, cam, mask, gb, base, row0 = ctx.saved_tensors
        V = planes.shape[1]
        g = grad_sp.float()
        if ctx.model_id == nat.MODEL_2DGS:
            # SP2 (u v opac M9 rgb ...) -> G_SP2 (du dv dM9 dopac drgb)
            gsp = torch.cat([g[:, 0:2], g[:, 3:12], g[:, 2:3], g[:, 12:15], torch.zeros_like(g[:, :1])],
                            1).contiguous()  # 16-float rows (include/splat_b200.h)
        else:
            gsp = g[:, :nat.GSP_FLOATS].contiguous()
        grad = torch.zeros_like(planes)
        desc = nat.ProjDesc(1, ctx.sh_degree, 0, 0, ctx.model_id, _CHUNK, 1)  # gsp_form 1: plain dL/dSP
        nat.call("bs_project_bwd", desc, nat.ptr(planes), V, nat.ptr(mask), nat.ptr(gb), ctx.ng, nat.ptr(base),
                 nat.ptr(row0), nat.ptr(cam), nat.ptr(gsp), nat.ptr(grad), nat.stream_handle())
        return grad, None, None, None, None


def pts_splatting(view: CameraView, PC: dict, infrustum_ids: torch.Tensor, sh_degree: int = 3,
                  model: str = "3dgs") -> dict:
    """Project the in-frustum points of PC into view-dependent splats (K1);
    differentiable with respect to the PC tensors (K1b)."""
    nat.load()
    model_id = _MODELS[model]
    ids = infrustum_ids.to(device=PC["xyz"].device, dtype=torch.int64)
    planes = pack_points(PC, ids)
    cam = _camera(view, planes.device)
    sp = _ProjectFn.apply(planes, cam, (view.width, view.height), sh_degree, model_id)
    if model_id == nat.MODEL_2DGS:
        return {"means2d": sp[:, 0:2], "opacities": sp[:, 2], "ray_transforms": sp[:, 3:12],
                "colors": sp[:, 12:15], "depths": sp[:, 15], "radii": sp[:, 16:18], "normals": sp[:, 18:21],
                "box_centers": sp[:, 22:24], "_model": model}
    return {"means2d": sp[:, 0:2], "opacities": sp[:, 2], "conics": sp[:, 3:6], "colors": sp[:, 6:9],
            "depths": sp[:, 9], "radii": sp[:, 10:12], "_model": model}


def pack_splats(SP: dict) -> torch.Tensor:
    """Differentiable inverse of the pts_splatting split: rows [V, SP]."""
    if SP.get("_model", "3dgs") == "2dgs":
        V = SP["means2d"].shape[0]
        pad = SP["means2d"].new_zeros(V, 1)
        # radii: half-widths of the support box centred at box_centers (binning, culling)
        cols = [SP["means2d"], SP["opacities"].reshape(-1, 1), SP["ray_transforms"], SP["colors"],
                SP["depths"].reshape(-1, 1).detach(), SP["radii"].detach(), SP["normals"].detach(), pad,
                SP["box_centers"].detach()]
    else:
        cols = [SP["means2d"], SP["opacities"].reshape(-1, 1), SP["conics"], SP["colors"],
                SP["depths"].reshape(-1, 1).detach(), SP["radii"].detach()]
    return torch.cat(cols, 1).float().contiguous()


# ---------------------------------------------------------------- image_render


class _RenderFn(torch.autograd.Function):
    """splat rows [V, SP] -> image [H, W, 3] (K2 + K3) / dL/dimage -> dL/drows (K4)."""

    @staticmethod
    def forward(ctx, rows, cam, W, H, bg, model_id):
        dev = rows.device
        V = rows.shape[0]
        tiles = ((W + 15) // 16) * ((H + 15) // 16)
        seg_row0 = torch.zeros(1, dtype=torch.int64, device=dev)
        seg_slot = torch.zeros(1, dtype=torch.int32, device=dev)
        buf = _Buffers()
        n_inst, irows, ranges, _ = bin_buckets(buf, rows, V, seg_row0, seg_slot, 1, cam, tiles, model_id)
        image = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
        final_T = torch.empty((H, W), dtype=torch.float32, device=dev)
        n_contrib = torch.empty((H, W), dtype=torch.int32, device=dev)
        desc = nat.RasterDesc(1, tiles, W, H, (ctypes.c_float * 3)(*bg), 0, 1)
        fwd, _ = _raster_names(model_id)
        nat.call(fwd, desc, nat.ptr(rows), nat.ptr(irows), nat.ptr(ranges), nat.ptr(image), nat.ptr(final_T),
                 nat.ptr(n_contrib), None, None, None, nat.stream_handle())
        ctx.save_for_backward(rows, irows[:max(n_inst, 1)].clone(), ranges.clone(), image, final_T, n_contrib)
        ctx.meta = (W, H, tuple(bg), model_id, tiles)
        return image

    @staticmethod
    def backward(ctx, grad_image):
        rows, irows, ranges, image, final_T, n_contrib = ctx.saved_tensors
        W, H, bg, model_id, tiles = ctx.meta
        gw = nat.GSP2_FLOATS if model_id == nat.MODEL_2DGS else nat.GSP_FLOATS
        g_sp = torch.zeros((rows.shape[0], gw), dtype=torch.float32, device=rows.device)
        desc = nat.RasterDesc(1, tiles, W, H, (ctypes.c_float * 3)(*bg), 0, 1)
        _, bwd = _raster_names(model_id)
        gimg = grad_image.float().contiguous()  # held until the launch is queued
        nat.call(bwd, desc, nat.ptr(rows), nat.ptr(irows), nat.ptr(ranges), nat.ptr(image), nat.ptr(final_T),
                 nat.ptr(n_contrib), nat.ptr(gimg), None, None, nat.ptr(g_sp), nat.stream_handle())
        grad_rows = torch.zeros_like(rows)
        if model_id == nat.MODEL_2DGS:
            grad_rows[:, 0:2] = g_sp[:, 0:2]
            # moments Ga, Gb, Gc of dL/dzeta (include/splat_b200.h) -> dL/dM rows
            r0, r1, r2 = rows[:, 3:6], rows[:, 6:9], rows[:, 9:12]
            ga, gb, gc = g_sp[:, 2:5], g_sp[:, 5:8], g_sp[:, 8:11]
            cr = torch.linalg.cross
            grad_rows[:, 3:6] = cr(r1, ga) + cr(gc, r2)
            grad_rows[:, 6:9] = cr(ga, r0) + cr(r2, gb)
            grad_rows[:, 9:12] = cr(gb, r1) + cr(r0, gc)
            grad_rows[:, 2] = g_sp[:, 11]
            grad_rows[:, 12:15] = g_sp[:, 12:15]
        else:
            # G_SP moments of dL/dpower (include/splat_b200.h) -> dL/d(u, v, conic)
            A, Bc, Cc = rows[:, 3], rows[:, 4], rows[:, 5]
            m1, m2 = g_sp[:, 0], g_sp[:, 1]
            grad_rows[:, 0] = -(A * m1 + Bc * m2)
            grad_rows[:, 1] = -(Bc * m1 + Cc * m2)
            grad_rows[:, 2] = g_sp[:, 2]
            grad_rows[:, 3] = -0.5 * g_sp[:, 3]
            grad_rows[:, 4] = -g_sp[:, 4]
            grad_rows[:, 5] = -0.5 * g_sp[:, 5]
            grad_rows[:, 6:9] = g_sp[:, 6:9]
        return grad_rows, None, None, None, None, None


def _raster_names(model_id):
    return ("bs_raster2d_fwd", "bs_raster2d_bwd") if model_id == nat.MODEL_2DGS else ("bs_raster_fwd",
                                                                                      "bs_raster_bwd")


def image_render(view: CameraView, SP: dict, bg=(0.0, 0.0, 0.0)) -> torch.Tensor:
    """Render all splats of SP into view (depth-sorted front-to-back alpha
    blending); differentiable with respect to the SP tensors."""
    nat.load()
    model_id = _MODELS[SP.get("_model", "3dgs")]
    rows = pack_splats(SP)
    cam = _camera(view, rows.device)
    return _RenderFn.apply(rows, cam, view.width, view.height, tuple(float(x) for x in bg), model_id)
