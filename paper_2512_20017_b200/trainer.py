"""Per-rank executor of one PBDR training step (Algorithm 1).

One process per GPU.  Rank k holds a shard PC_k of the Z-ordered point cloud
(whole point groups, ascending global index) in the plane-major parameter
layout of include/splat_b200.h plus its Adam moments.  A step over a batch
of views runs, all on the GPU through the C ABI:

  K0  bs_cull_count(MASK)        pts_culling for every batch view (line 3)
      -> C[v]_k per view          (line 4)
  [N>1] all_gather C -> A; host hierarchical_place -> W   (lines 6-8)
      bs_scan_counts             SP row layout in destination order
  K1  bs_project_fwd             pts_splatting (line 5) straight into the
                                 all-to-all send layout
  [N>1] all_to_all_single SP     (line 9)
  K2  depth keys + radix sort + tile count/emit + radix sort + ranges
  K3  bs_raster_fwd (+ fused mean-L1 loss partials)     (lines 11-15)
  K4  bs_raster_bwd (L1 gradient recomputed in-kernel)  (lines 17-19)
      3DGS: K3 + L + K4 as one kernel, bs_raster_fwd_bwd (each warp keeps
      its forward's splat list in shared memory for the backward)
  [N>1] reverse all_to_all_single G_SP                  (line 21)
  K1b+K5 bs_project_bwd_adam      (lines 22-27), fused per point

There is no CPU path: every kernel call raises if the library or the GPU is
missing.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .binning import bin_buckets
from .culling import view_plane_block
from .exchange import layout_for
from .scenes import CameraView

_CAM_BYTES = ctypes.sizeof(nat.Camera)
_NVTX = os.environ.get("BS_NVTX", "0") == "1"


def camera_struct(view: CameraView) -> nat.Camera:
    fx, fy, cx, cy = view.intrinsics()
    c = nat.Camera()
    rot_cw = np.asarray(view.rotation, dtype=np.float64).T.astype(np.float32).reshape(9)
    for k in range(9):
        c.rot_cw[k] = float(rot_cw[k])
    for k in range(3):
        c.pos[k] = float(np.float32(view.position[k]))
    c.fx, c.fy, c.cx, c.cy = fx, fy, cx, cy
    c.lim_x = 1.3 * math.tan(view.fov_x / 2.0)
    c.lim_y = 1.3 * math.tan(view.fov_y / 2.0)
    c.near_plane, c.far_plane = view.near, view.far
    c.width, c.height = view.width, view.height
    return c


def camera_bytes(views) -> np.ndarray:
    buf = bytearray()
    for v in views:
        buf += bytes(camera_struct(v))
    return np.frombuffer(bytes(buf), dtype=np.uint8).reshape(len(views), _CAM_BYTES).copy()


@dataclass
class AdamConfig:
    lr: np.ndarray  # (60,) per-lane learning rates
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15
    selective: bool = False


@dataclass
class DensifyConfig:
    """Periodic densification (standard 3DGS clone / split /
    prune, include/splat_b200.h bs_densify_*).  grad_threshold: on the mean
    NDC-space |dL/d mean2d| since the last densification (3DGS: 2e-4);
    split_scale: points whose largest world scale exceeds it are split in
    two, the others cloned (3DGS: 0.01 x the scene extent); min_opacity:
    prune below (3DGS: 0.005); max_scale: also prune points larger than this
    (0: off); seed: the split samples (keyed by global point id)."""

    grad_threshold: float = 2e-4
    split_scale: float = 0.01
    min_opacity: float = 0.005
    max_scale: float = 0.0
    seed: int = 0


class _Grow:
    """Grow-only cache of device buffers keyed by name."""

    def __init__(self, dev):
        self.dev = dev
        self.bufs = {}

    def get(self, name, n, dtype):
        b = self.bufs.get(name)
        if b is None or b.numel() < n or b.dtype != dtype:
            cap = max(int(n * 1.25) + 1024, 1024)
            b = torch.empty(cap, dtype=dtype, device=self.dev)
            self.bufs[name] = b
        return b[:n]


def _bits_for(n: int) -> int:
    return max(1, int(math.ceil(math.log2(max(n, 2)))))


class SplatTrainer:
    """Rank-local state + one training step.  `params` is the plane-major
    [15, S, 4] float32 shard (ascending global point index); `group_begin`
    (int32, n_groups+1) and `aabb` (float32, n_groups x 6) describe its point
    groups; `views` are all dataset views (the batch picks from them);
    `gt` is u8 [n_views, H, W, 3] (device-resident ground truth);
    `global_ids` (int [S], ascending) the global point index of every shard
    point (default: the local index, i.e. a single rank holding every point).
    With several ranks the received splat rows of every rendered view are put
    in ascending global-id order before binning (bs_canonical_order), so the
    per-tile lists are the single-rank lists on any number of ranks."""

    def __init__(self, params: np.ndarray, group_begin: np.ndarray, aabb: np.ndarray, views, gt=None,
                 sh_degree: int = 3, adam: AdamConfig | None = None, device=None, comm=None,
                 bg=(0.0, 0.0, 0.0), model: str = "3dgs", presence: np.ndarray | None = None,
                 gt_view_ids=None, patches: int = 1, global_ids: np.ndarray | None = None):
        nat.load()
        if model not in ("3dgs", "2dgs"):
            raise ValueError(f"unknown splat model {model!r} (3dgs | 2dgs)")
        self.model = model
        self.model_id = nat.MODEL_2DGS if model == "2dgs" else nat.MODEL_3DGS
        self.sp_floats = nat.SP2_FLOATS if model == "2dgs" else nat.SP_FLOATS
        self.gsp_floats = nat.GSP2_FLOATS if model == "2dgs" else nat.GSP_FLOATS
        self.gsp_wire_floats = 15 if model == "2dgs" else 9  # floats of a G_SP row that carry data
        self._raster = ("bs_raster2d_fwd", "bs_raster2d_bwd") if model == "2dgs" else ("bs_raster_fwd",
                                                                                      "bs_raster_bwd")
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.S = int(params.shape[1])
        self.params = torch.as_tensor(np.ascontiguousarray(params, dtype=np.float32), device=self.dev)
        self.exp_avg = torch.zeros_like(self.params)
        self.exp_avg_sq = torch.zeros_like(self.params)
        self.group_begin = torch.as_tensor(np.asarray(group_begin, dtype=np.int32), device=self.dev)
        self.aabb = torch.as_tensor(np.ascontiguousarray(aabb, dtype=np.float32).reshape(-1, 6), device=self.dev)
        self.n_groups = len(group_begin) - 1
        gsz = np.diff(np.asarray(group_begin, dtype=np.int64))
        self.max_group = int(gsz.max()) if len(gsz) else 0  # per-point kernels: one CTA per 256 points
        self.max_chunks = max(1, -(-self.max_group // 256))
        self.views = list(views)
        self.W, self.H = self.views[0].width, self.views[0].height
        if any((v.width, v.height) != (self.W, self.H) for v in self.views):
            raise ValueError("all views of a trainer must share one image size")
        self.tiles_x = (self.W + nat.TILE - 1) // nat.TILE
        self.tiles_y = (self.H + nat.TILE - 1) // nat.TILE
        self.tiles = self.tiles_x * self.tiles_y
        # patches per image side: with several ranks each of the B P^2 patches
        # of a batch is placed on its own; one rank renders
        # whole views whatever P is
        if not (1 <= int(patches) <= 8):
            raise ValueError("patches (P) must be in [1, 8]")
        self.P = int(patches)
        self.planes_all = torch.as_tensor(np.stack([view_plane_block(v, self.P) for v in self.views]),
                                          device=self.dev)
        self.cams_all = torch.as_tensor(camera_bytes(self.views), device=self.dev)
        # 4DGS spatio-temporal culling (visibility.py:244-252):
        # point i is a candidate for view v iff presence[i, 0] <= t_v <= presence[i, 1] (f32)
        self.global_ids = None
        if global_ids is not None:
            gid = np.asarray(global_ids, dtype=np.int64)
            if gid.shape != (self.S,) or (len(gid) and (np.any(np.diff(gid) <= 0) or gid[0] < 0 or gid[-1] >= 2**31)):
                raise ValueError("global_ids must be ascending int32-range point indices, one per shard point")
            self.global_ids = torch.as_tensor(gid.astype(np.int32), device=self.dev)
        self.record_row_gid = False  # single rank: also write the rows' global ids (tests)
        # see _use_work (BS_CHUNK_LIST=0/1 forces it: tuning experiments)
        self.visible_chunk_list = {"0": False, "1": True}.get(os.environ.get("BS_CHUNK_LIST", ""), "auto")
        # the fused raster's per-pixel transmittance / contributor count
        # (last["final_T"], last["n_contrib"]): not needed by the step, written
        # only when asked for (8 B per pixel; the separate kernels always write them)
        self.keep_raster_aux = False
        self._last_fill, self._work_on = 0.0, False
        self.presence = self.view_times = None
        if presence is not None:
            pres = np.ascontiguousarray(presence, dtype=np.float32)
            if pres.shape != (self.S, 2):
                from .status import ParameterError

                raise ParameterError("presence must be float32 [S, 2] aligned with the shard")
            if any(v.time is None for v in self.views):
                from .status import ConfigurationError

                raise ConfigurationError("temporal culling needs a timestamp on every view")
            self.presence = torch.as_tensor(pres, device=self.dev)
            self.view_times = torch.as_tensor(np.array([v.time for v in self.views], dtype=np.float32),
                                              device=self.dev)
        self.gt = None if gt is None else torch.as_tensor(gt, device=self.dev)
        # gt_view_ids: the view id of each row of `gt` when it holds a subset
        self.gt_lut = None
        if gt_view_ids is not None:
            lut = np.full(len(self.views), -1, dtype=np.int32)
            lut[np.asarray(gt_view_ids, dtype=np.int64)] = np.arange(len(gt_view_ids), dtype=np.int32)
            self.gt_lut = torch.as_tensor(lut, device=self.dev)
        self.sh_degree = sh_degree
        self.adam = adam if adam is not None else AdamConfig(np.full(60, 1e-3, dtype=np.float32))
        self.step_count = 0
        self.comm = comm
        self.bg = bg
        self.buf = _Grow(self.dev)
        self.timers = None  # optional {stage: [(start_evt, end_evt), ...]}
        self.last = {}
        self.binning = "bucket"  # or "radix" (identical lists, see csrc/bin_tiles.cu)
        # single rank: the projection counts the tile buckets (no count pass)
        self.single_pass_bin = os.environ.get("BS_SINGLE_PASS_BIN", "1") == "1"
        self.sort_cap = 16384    # bucket sizes sorted in shared memory
        self.bin_capacity_hint = None  # initial instance-key buffer (tests of the overflow re-run)
        # raster work split: pixels per lane (1 -> 8x4 region per warp, 2 -> 8x8);
        # 1 measured faster on B200 (C2: bwd 3.30 vs 3.52 ms, fwd 1.22 vs 1.24 ms)
        self.pixels_per_lane = int(os.environ.get("BS_RASTER_PPL", "1"))
        # 3DGS mean-L1 step: forward + loss + backward in one kernel (bs_raster_fwd_bwd)
        self.raster_fused = os.environ.get("BS_RASTER_FUSED", "1") == "1"
        # densification statistic (track_densify_stats): float2 per point
        self.densify_stats = None
        # a stable global key per local group (first global id at construction):
        # orders the groups of all ranks when densification renumbers the points
        gb0 = np.asarray(group_begin, dtype=np.int64)[:-1]
        if self.global_ids is not None and self.S:
            keys = np.asarray(global_ids, dtype=np.int64)[np.minimum(gb0, self.S - 1)]
        else:
            keys = gb0.copy()
        self.group_keys = keys
        # per-view device tables the batch's rows are selected from (the view
        # ids travel as kernel parameters: csrc/views.cu)
        self._gt_index = (self.gt_lut if self.gt_lut is not None
                          else torch.arange(len(self.views), dtype=torch.int32, device=self.dev))
        # N = 1: the splat buffer is sized for every point in every batch view
        # when that fits this budget, so the projection is launched before the
        # host reads the row counts (the read then overlaps the projection)
        self.sp_capacity_bytes = 2 << 30
        self._rows_pin = torch.empty(32, dtype=torch.int64, pin_memory=True)

    # ------------------------------------------------------------------ utils
    def _t(self, name):
        """Context manager around a stage: CUDA events (if `timers` is
        enabled) and an NVTX range named after the stage (if BS_NVTX=1, for
        nsys / ncu --nvtx; SURVEY.md §5 tracing)."""
        trainer = self

        class _T:
            def __enter__(self_):
                if _NVTX:
                    torch.cuda.nvtx.range_push(f"bs:{name}")
                if trainer.timers is not None:
                    self_.s = torch.cuda.Event(enable_timing=True)
                    self_.s.record()
                return self_

            def __exit__(self_, *exc):
                if trainer.timers is not None:
                    e = torch.cuda.Event(enable_timing=True)
                    e.record()
                    trainer.timers.setdefault(name, []).append((self_.s, e))
                if _NVTX:
                    torch.cuda.nvtx.range_pop()
                return False

        return _T()

    # ------------------------------------------------------------------ step
    def _work_list(self):
        return self.buf.get("work_list", max(self.n_groups * self.max_chunks, 1), torch.int32)

    def _work_count(self):
        return self.buf.get("work_count", 1, torch.int32)

    def _use_work(self):
        """Visible-chunk work list (culling -> projection kernels): on when the
        previous step projected under half of its (point, view) pairs -- a
        sparse step (C4: ~2 %), where one CTA per (group, chunk) mostly
        launches empty CTAs; off for dense steps (C2: every point in every
        view), where the listing and the shuffled chunk order cost ~20 us.
        `visible_chunk_list` = True / False forces it.  Same results."""
        if self.visible_chunk_list != "auto":
            return bool(self.visible_chunk_list)
        return self._last_fill < 0.5

    def _set_work(self, pdesc):
        """Projection descriptor: visit only the chunks the step's culling listed."""
        if self.max_group > 0 and self._work_on:
            pdesc.work_list, pdesc.work_count = nat.ptr(self._work_list()), nat.ptr(self._work_count())

    def _up(self, arr, name, dtype):
        """Small per-step host table -> reused device buffer (bs_upload: no
        copy engine, no stream synchronisation)."""
        a = np.ascontiguousarray(arr, dtype={torch.int64: np.int64, torch.int32: np.int32}[dtype])
        return nat.upload(a, self.buf.get(name, max(a.size, 1), dtype)[: a.size])

    def _wait_gt(self):
        """The compute stream waits for the caller's ground-truth upload (once)."""
        if getattr(self, "_gt_ready", None) is not None:
            torch.cuda.current_stream().wait_event(self._gt_ready)
            self._gt_ready = None

    def _select_views(self, ids, table, name):
        """Rows `ids` (host view indices, <= 32) of a per-view device table,
        into a reused device buffer: bs_select_rows passes the ids as kernel
        parameters, so nothing waits on a copy engine (csrc/views.cu)."""
        n = len(ids)
        row = table[0].numel()
        out = self.buf.get(name, max(n, 1) * row, table.dtype)[: n * row].view(n, *table.shape[1:])
        ids32 = np.ascontiguousarray(ids, dtype=np.int32)
        nat.call("bs_select_rows", ids32.ctypes.data, n, nat.ptr(table), table.shape[0], row * table.element_size(),
                 nat.ptr(out), nat.stream_handle())
        return out


    def _cull_counts(self, batch_ids, mask, counts, base, view_rows, view_row0, st, patch_counts=None,
                     chunk_prefix=None, tag=""):
        B = len(batch_ids)
        planes = self._select_views(batch_ids, self.planes_all, "planes_sel" + tag)
        temporal = self.presence is not None
        times = self._select_views(batch_ids, self.view_times, "times_sel" + tag) if temporal else None
        desc = nat.CullDesc(nat.CULL_MASK, B, self.P, 1, 1 if temporal else 0, 4, self.max_chunks, nat.ptr(chunk_prefix))
        if not tag:
            self._work_on = chunk_prefix is not None and self.max_group > 0 and self._use_work()
        nat.call("bs_cull_count", desc, nat.ptr(self.params), self.S, nat.ptr(self.presence),
                 nat.ptr(self.group_begin), nat.ptr(self.aabb), self.n_groups, nat.ptr(planes), nat.ptr(times),
                 None, nat.ptr(mask), nat.ptr(counts), nat.ptr(patch_counts), st)
        order = np.arange(B, dtype=np.int32)
        nat.call("bs_scan_counts", nat.ptr(counts), self.n_groups, B, order.ctypes.data, nat.ptr(base),
                 nat.ptr(view_rows), nat.ptr(view_row0), st)
        if not tag and self._work_on:
            # the chunks with a visible point, for the projection kernels'
            # grid-stride loops (bs_proj_desc.work_list)
            nat.call("bs_list_chunks", nat.ptr(counts), nat.ptr(chunk_prefix), nat.ptr(self.group_begin),
                     self.n_groups, self.max_chunks, B, nat.ptr(self._work_list()), nat.ptr(self._work_count()), st)

    def step(self, batch_ids, gt_batch: torch.Tensor | None = None, next_batch=None, gt_ready=None):
        """One training step over `batch_ids` (indices into self.views).
        Returns the mean-L1 losses of the views rendered on THIS rank as a
        device tensor, in batch order (N = 1: all B views); their batch
        positions are in self.last["loss_views"] (with several ranks each
        rank returns its own views' losses, W of PAPER.md:488).
        With several ranks, `next_batch` (the same on every rank) starts the
        asynchronous placement of the following step (exchange.py).
        `gt_ready` (optional CUDA event): `gt_batch` is being uploaded on
        another stream; the step waits for it only where the ground truth is
        first read (the raster), so the upload overlaps culling, projection
        and binning."""
        B = len(batch_ids)
        self._gt_ready = gt_ready
        if not (1 <= B <= 32):
            raise ValueError("batch must hold 1..32 views")
        dev, S, st = self.dev, self.S, nat.stream_handle()
        cams = self._select_views(batch_ids, self.cams_all, "cams_sel")
        # ---- K0: culling -> visibility masks + per-(group, view) counts
        mask = self.buf.get("mask", S, torch.int32)
        counts = self.buf.get("counts", self.n_groups * B, torch.int32)
        base = self.buf.get("base", self.n_groups * B, torch.int32)
        view_rows = self.buf.get("view_rows", B, torch.int64)
        view_row0 = self.buf.get("view_row0", B, torch.int64)
        patched = self.comm is not None and self.P > 1
        patch_counts = self.buf.get("patch_counts", B * self.P * self.P, torch.int64) if patched else None
        # rows of each (group, 256-point chunk) before the chunk, for the projection kernels
        chunk_prefix = self.buf.get("chunk_prefix", self.n_groups * self.max_chunks * B, torch.int32)
        with self._t("cull"):
            self._cull_counts(batch_ids, mask, counts, base, view_rows, view_row0, st, patch_counts,
                              chunk_prefix)
        if self.comm is not None and next_batch is not None:
            # counts of the next batch (per view, or per patch when P > 1) on
            # the pre-update positions -> its W on a host thread (exchange.py)
            Bn = len(next_batch)
            nb = self.buf
            pc_next = nb.get("patch_counts_next", Bn * self.P * self.P, torch.int64) if patched else None
            self._cull_counts(next_batch, nb.get("mask_next", S, torch.int32),
                              nb.get("counts_next", self.n_groups * Bn, torch.int32),
                              nb.get("base_next", self.n_groups * Bn, torch.int32),
                              nb.get("view_rows_next", Bn, torch.int64), nb.get("view_row0_next", Bn, torch.int64), st,
                              patch_counts=pc_next, tag="_next")
            self.comm.prefetch(pc_next if patched else nb.get("view_rows_next", Bn, torch.int64),
                               tuple(int(v) for v in next_batch))
        if patched:
            return self._step_patches(batch_ids, gt_batch, cams, mask, base, view_rows, view_row0,
                                      patch_counts, st, chunk_prefix)
        lay = None
        pdesc = nat.ProjDesc(B, self.sh_degree, self.tiles_x, self.tiles_y, self.model_id, self.max_group, 0,
                             nat.ptr(chunk_prefix))
        pdesc.point_gid = nat.ptr(self.global_ids)
        pdesc.densify_stats = nat.ptr(self.densify_stats)
        self._set_work(pdesc)
        early = self.comm is None and S * B * self.sp_floats * 4 <= self.sp_capacity_bytes
        row_gid = None
        if self.comm is not None or self.record_row_gid:
            row_gid = self.buf.get("row_gid", max(S * B, 1), torch.int32)
            pdesc.row_gid = nat.ptr(row_gid)
        support = records = None
        if self.comm is None:
            # the rasterisers' per-row support threshold, written with the rows
            support = self.buf.get("row_support", max(S * B, 1), torch.float32)
            pdesc.row_support = nat.ptr(support)
            if early and self.binning != "radix" and self.single_pass_bin:
                # single-pass binning: the projection counts the (view, tile)
                # buckets and records each row's tile rectangle
                records = self._single_pass_bin(pdesc, B, S * B)
        if early:
            # the row counts start towards the host before the projection is
            # queued, so the host resumes while the projection still runs
            rows_pin = self._rows_pin[:B]
            nat.call("bs_copy_to_host", nat.ptr(view_rows), 8 * B, rows_pin.data_ptr(), st)
            rows_ready = torch.cuda.Event()
            rows_ready.record()
            # ---- K1 first (rows land at view_row0 from the scan), then the
            # row counts are read while the projection runs
            sp = self.buf.get("sp", max(S * B, 1) * self.sp_floats, torch.float32)
            if self.binning != "radix" and self.model == "3dgs":
                # single rank: the projection clears the G_SP accumulator rows
                # as it writes the SP rows (no separate clearing pass; C2 -24 us
                # per step, measured a wash for the 64-byte 2DGS rows)
                pdesc.gsp_zero = nat.ptr(self.buf.get("gsp", max(S * B, 1) * self.gsp_floats, torch.float32))
            with self._t("project"):
                nat.call("bs_project_fwd", pdesc, nat.ptr(self.params), S, nat.ptr(mask),
                         nat.ptr(self.group_begin), self.n_groups, nat.ptr(base), nat.ptr(view_row0), nat.ptr(cams),
                         nat.ptr(sp), st)
        if early:
            rows_ready.synchronize()  # C[v]_k (sync 1: sizes the render buffers)
            rows_host = rows_pin.numpy().copy()
        elif self.comm is None:
            rows_host = view_rows.cpu().numpy()
        else:
            # A <- all-gather C[.]_k ; W <- AssignImages(A)  (Alg. 1 lines 6-8)
            with self._t("assign"):
                A = self.comm.gather_access(view_rows)
                W = self.comm.assign(A, key=tuple(int(v) for v in batch_ids))
                lay = layout_for(A, W, self.comm.rank)
                rows_host = A[:, self.comm.rank].copy()
                row0 = np.zeros(B, dtype=np.int64)
                row0[lay.order] = np.concatenate([[0], np.cumsum(rows_host[lay.order])[:-1]])
                nat.upload(row0, view_row0)
            self.last.update(A=A, W=W, layout=lay)
        n_rows = int(rows_host.sum())
        self._last_fill = n_rows / max(1, S * B)
        self.last["rows_per_view"] = rows_host.copy()
        peer = None
        if lay is not None and getattr(self.comm, "peer", False):
            # peer-memory exchange: the projection writes every row straight
            # into its renderer's receive buffer (exchange.PeerExchange)
            peer = self.comm.plan(lay, self.sp_floats, self.gsp_floats)
            pdesc.view_sp, pdesc.view_gid = nat.ptr(peer["view_sp"]), nat.ptr(peer["view_gid"])
            pdesc.row_gid = None
        if not early:
            # ---- K1: projection into SP rows (send layout)
            if self.comm is None and self.binning != "radix" and self.single_pass_bin:
                records = self._single_pass_bin(pdesc, B, n_rows)  # sized by the row counts just read
            sp = self.buf.get("sp", max(n_rows, 1) * self.sp_floats, torch.float32)
            with self._t("project"):
                nat.call("bs_project_fwd", pdesc, nat.ptr(self.params), S, nat.ptr(mask),
                         nat.ptr(self.group_begin), self.n_groups, nat.ptr(base), nat.ptr(view_row0), nat.ptr(cams),
                         nat.ptr(sp), st)
        if lay is None:
            # every batch view is rendered here (N = 1: W[v] = k for all v):
            # one segment per view, starting at the scan's view_row0; the rows
            # of a view are in ascending point order, the canonical order
            if row_gid is not None:
                self.last["row_gid"] = row_gid[:n_rows]
            seg_row0 = view_row0
            seg_slot = self._slot_ids(B)
            self.last["loss_views"] = list(range(B))
            losses, gsp = self._render_and_backward(sp, n_rows, seg_row0, seg_slot, B, cams, batch_ids, gt_batch,
                                                    gsp_cleared=bool(pdesc.gsp_zero), support=support,
                                                    records=records)
        else:
            # SP all-to-all to the rendering ranks (line 9), render, G_SP back (line 21)
            with self._t("a2a_fwd"):
                if peer is not None:
                    self.comm.forward_done(lay, self.sp_floats, st)
                    sp_recv, gid_recv = peer["sp_recv"], peer["gid_recv"]
                else:
                    sp_recv = self.comm.forward(sp[: n_rows * self.sp_floats], lay, self.sp_floats).reshape(-1)
                    gid_recv = self.comm.forward_ids(row_gid[:n_rows], lay)
            mine = self._up(lay.my_views, "mine", torch.int64)
            n_slots = len(lay.my_views)
            self.last["loss_views"] = [int(v) for v in lay.my_views]
            # received rows in canonical order: per rendered view, ascending global id
            slot_rows = np.bincount(lay.seg_slot, weights=lay.seg_rows, minlength=n_slots).astype(np.int64)
            sp_c, order = self._canonical(sp_recv, gid_recv, lay.n_recv, lay.seg_rows, lay.seg_slot, n_slots)
            seg_row0 = self._up(np.concatenate([[0], np.cumsum(slot_rows)[:-1]]), "seg_row0", torch.int64)
            seg_slot = self._slot_ids(n_slots)
            gt_slots = None
            if gt_batch is not None:
                self._wait_gt()
                gt_slots = gt_batch.index_select(0, mine).contiguous()
            losses, gsp_c = self._render_and_backward(sp_c, lay.n_recv, seg_row0, seg_slot, n_slots,
                                                      cams.index_select(0, mine).contiguous(),
                                                      [batch_ids[int(m)] for m in lay.my_views], gt_slots,
                                                      support=self._recv_support)
            with self._t("a2a_bwd"):
                wire = self.gsp_wire_floats
                if peer is not None:
                    # each canonical row straight into its owner's send-layout slot
                    seg_row0_r = self._up(np.concatenate([[0], np.cumsum(lay.seg_rows)[:-1]]), "seg_row0_r",
                                          torch.int64)
                    nat.call("bs_return_rows", nat.ptr(gsp_c), self.gsp_floats, wire, nat.ptr(order), lay.n_recv,
                             nat.ptr(seg_row0_r), nat.ptr(peer["seg_src"]), nat.ptr(peer["seg_dst0"]), peer["n_segs"],
                             nat.ptr(peer["dst"]), self.gsp_floats, st)
                    self.comm.backward_done(lay, wire, st)
                    gsp = peer["gsp_home"]
            if peer is None:
                with self._t("a2a_bwd"):
                    # back to the received order, only the used floats of a G_SP
                    # row (3DGS: 9 of the 12), then to the owners
                    g = self._uncanonical(gsp_c, order, lay.n_recv, wire)
                    back = self.comm.backward(g, lay, wire).view(-1, wire)
                    if wire != self.gsp_floats:
                        full = self.buf.get("gsp_home", max(back.shape[0], 1) * self.gsp_floats, torch.float32)
                        full = full[: back.shape[0] * self.gsp_floats].view(-1, self.gsp_floats)
                        full.zero_()
                        full[:, :wire] = back
                        back = full
                    gsp = back.reshape(-1)
        # ---- K1b + K5: projection backward fused with Adam
        self.step_count += 1
        ad = nat.AdamDesc()
        for k in range(60):
            ad.lr[k] = float(self.adam.lr[k])
        ad.beta1, ad.beta2, ad.eps = self.adam.beta1, self.adam.beta2, self.adam.eps
        ad.step, ad.selective = self.step_count, 1 if self.adam.selective else 0
        with self._t("project_bwd_adam"):
            nat.call("bs_project_bwd_adam", pdesc, ad, nat.ptr(self.params), nat.ptr(self.exp_avg),
                     nat.ptr(self.exp_avg_sq), S, nat.ptr(mask), nat.ptr(self.group_begin), self.n_groups,
                     nat.ptr(base), nat.ptr(view_row0), nat.ptr(cams), nat.ptr(gsp), st)
        return losses

    def _step_patches(self, batch_ids, gt_batch, cams, mask, base, view_rows, view_row0, patch_counts, st,
                      chunk_prefix=None):
        """Alg. 1 with P x P patches per view on several ranks (SURVEY.md
        §8(e)): A over the B P^2 patches -> W; every rank projects its points
        for all batch views, sends each splat row to the ranks whose patches
        its support reaches (csrc/patches.cu; the render set, a superset of
        A), renders only the pixels of its own patches, and the returned
        gradient rows are summed into the rows they came from."""
        comm, P = self.comm, self.P
        B, N, me, PP = len(batch_ids), self.comm.world, self.comm.rank, self.P * self.P
        dev, S = self.dev, self.S
        with self._t("assign"):
            A = comm.gather_access(patch_counts)       # int64 [B P^2, N]
            W = comm.assign(A, key=tuple(int(v) for v in batch_ids))  # patch -> rank (prefetched when given)
        rows_host = view_rows.cpu().numpy()
        n_rows = int(rows_host.sum())
        self._last_fill = n_rows / max(1, S * B)
        self.last.update(A=A, W=W, rows_per_view=rows_host.copy())
        sp = self.buf.get("sp", max(n_rows, 1) * self.sp_floats, torch.float32)
        pdesc = nat.ProjDesc(B, self.sh_degree, self.tiles_x, self.tiles_y, self.model_id, self.max_group, 0,
                             nat.ptr(chunk_prefix))
        pdesc.densify_stats = nat.ptr(self.densify_stats)
        self._set_work(pdesc)
        row_gid = self.buf.get("row_gid", max(n_rows, 1), torch.int32)
        pdesc.point_gid, pdesc.row_gid = nat.ptr(self.global_ids), nat.ptr(row_gid)
        with self._t("project"):
            nat.call("bs_project_fwd", pdesc, nat.ptr(self.params), S, nat.ptr(mask), nat.ptr(self.group_begin),
                     self.n_groups, nat.ptr(base), nat.ptr(view_row0), nat.ptr(cams), nat.ptr(sp), st)
        # ---- render sets -> send layout (destination, view, row)
        owner = self._up(W, "owner", torch.int32)
        dmask = self.buf.get("dest_mask", max(n_rows, 1), torch.int32)
        nat.call("bs_row_dest_mask", nat.ptr(sp), self.model_id, n_rows, nat.ptr(view_row0), B, P, self.W, self.H,
                 nat.ptr(owner), nat.ptr(dmask), st)
        lib = nat.load()
        ws = self.buf.get("dest_ws", lib.bs_dest_compact_workspace(max(n_rows, 1), N), torch.uint8)
        totals = self.buf.get("dest_total", N, torch.int64)
        nat.call("bs_dest_compact", nat.ptr(dmask), n_rows, N, nat.ptr(view_row0), B, 1, nat.ptr(totals), None, None,
                 None, nat.ptr(ws), ws.numel(), st)
        send_rows = [int(x) for x in totals.cpu().tolist()]
        n_send = sum(send_rows)
        base_d = self._up(np.concatenate([[0], np.cumsum(send_rows)[:-1]]), "base_d", torch.int64)
        send_idx = self.buf.get("send_idx", max(n_send, 1), torch.int64)
        vcounts = self.buf.get("dest_view_counts", N * B, torch.int64)
        vcounts.zero_()
        nat.call("bs_dest_compact", nat.ptr(dmask), n_rows, N, nat.ptr(view_row0), B, 0, nat.ptr(totals),
                 nat.ptr(base_d), nat.ptr(send_idx), nat.ptr(vcounts), nat.ptr(ws), ws.numel(), st)
        recv_v = comm.exchange_counts(vcounts.view(N, B))   # [source, view] rows coming here
        recv_rows = [int(x) for x in recv_v.sum(axis=1)]
        send_sp = self.buf.get("send_sp", max(n_send, 1) * self.sp_floats, torch.float32)
        nat.call("bs_gather_rows", nat.ptr(sp), self.sp_floats, nat.ptr(send_idx), n_send, nat.ptr(send_sp), st)
        send_gid = self.buf.get("send_gid", max(n_send, 1), torch.int32)
        nat.call("bs_gather_rows", nat.ptr(row_gid), 1, nat.ptr(send_idx), n_send, nat.ptr(send_gid), st)
        with self._t("a2a_fwd"):
            sp_recv = comm._a2a(send_sp[: n_send * self.sp_floats], send_rows, recv_rows, self.sp_floats)
            gid_recv = comm._a2a(send_gid[:n_send], send_rows, recv_rows, 1).view(-1)
        comm.bytes_fwd += (n_send - send_rows[me]) * (self.sp_floats + 1) * 4
        # ---- render the own patches of every view that has one here
        Wm = np.asarray(W, dtype=np.int64).reshape(B, PP)
        my_views = [v for v in range(B) if (Wm[v] == me).any()]
        slot_bits = np.array([int(sum(1 << j for j in range(PP) if Wm[v, j] == me)) for v in my_views],
                             dtype=np.uint64)
        seg_rows, seg_slot = [], []
        for s_ in range(N):
            for k, v in enumerate(my_views):
                seg_rows.append(int(recv_v[s_, v]))
                seg_slot.append(k)
        n_recv = int(sum(recv_rows))
        self.last.update(my_views=my_views, send_rows=send_rows, recv_rows=recv_rows, n_send=n_send,
                         loss_views=list(my_views))
        losses = torch.zeros(0, dtype=torch.float32, device=dev)
        wire = self.gsp_wire_floats
        g = self.buf.get("gsp_wire", max(n_recv, 1) * wire, torch.float32)[: n_recv * wire]
        if my_views:
            n_slots = len(my_views)
            mine = self._up(my_views, "mine", torch.int64)
            # canonical order of the received rows (per slot, ascending global id)
            sp_c, order = self._canonical(sp_recv.reshape(-1), gid_recv, n_recv, seg_rows, seg_slot, n_slots)
            slot_rows = np.bincount(np.asarray(seg_slot), weights=np.asarray(seg_rows), minlength=n_slots)
            seg_row0 = self._up(np.concatenate([[0], np.cumsum(slot_rows)[:-1]]), "seg_row0", torch.int64)
            bits_t = self._up(slot_bits.view(np.int64), "slot_bits", torch.int64)
            if gt_batch is not None:
                self._wait_gt()
            gt_slots = gt_batch.index_select(0, mine).contiguous() if gt_batch is not None else None
            losses, gsp_c = self._render_and_backward(sp_c, n_recv, seg_row0, self._slot_ids(n_slots), n_slots,
                                                      cams.index_select(0, mine).contiguous(),
                                                      [batch_ids[int(m)] for m in my_views], gt_slots,
                                                      slot_patches=bits_t,
                                                      support=self._recv_support)
            g = self._uncanonical(gsp_c, order, n_recv, wire)
        # ---- gradient rows back to their sources, summed into the row they left
        with self._t("a2a_bwd"):
            back = comm._a2a(g.reshape(-1), recv_rows, send_rows, wire)
        comm.bytes_bwd += (n_recv - recv_rows[me]) * wire * 4
        gsp = self.buf.get("gsp_home", max(n_rows, 1) * self.gsp_floats, torch.float32)
        gsp.zero_()
        nat.call("bs_scatter_add_rows", nat.ptr(back), wire, wire, nat.ptr(send_idx), n_send, nat.ptr(gsp),
                 self.gsp_floats, st)
        self.step_count += 1
        ad = self._adam_desc()
        with self._t("project_bwd_adam"):
            nat.call("bs_project_bwd_adam", pdesc, ad, nat.ptr(self.params), nat.ptr(self.exp_avg),
                     nat.ptr(self.exp_avg_sq), S, nat.ptr(mask), nat.ptr(self.group_begin), self.n_groups,
                     nat.ptr(base), nat.ptr(view_row0), nat.ptr(cams), nat.ptr(gsp), st)
        return losses

    # ------------------------------------------------------------------ densification
    def track_densify_stats(self, on: bool = True) -> None:
        """Accumulate the densification statistic in every step's fused
        projection backward (3DGS): per point, the NDC-space |dL/d mean2d| of
        each batch view with a valid splat, and the number of such views."""
        if on and self.model != "3dgs":
            from .status import ParameterError

            raise ParameterError("densification is implemented for the 3DGS model")
        self.densify_stats = torch.zeros(max(self.S, 1), 2, dtype=torch.float32, device=self.dev) if on else None

    def densify(self, cfg: DensifyConfig | None = None) -> dict:
        """Clone / split / prune this rank's shard on the GPU (bs_densify_mark
        -> scan -> bs_densify_apply -> bs_group_aabb_ranges) from the
        statistic accumulated since the last call, then reset it.  Points stay
        in their groups, so the partition and the culling structures keep
        working; with several ranks (collective) the points are renumbered in
        global group order so the global ids -- and the canonical per-tile
        order -- are the single-rank ones.  Returns the action counts."""
        from .status import ParameterError

        if self.model != "3dgs":
            raise ParameterError("densification is implemented for the 3DGS model")
        cfg = cfg if cfg is not None else DensifyConfig()
        st = nat.stream_handle()
        S, ng, dev = self.S, self.n_groups, self.dev
        desc = nat.DensifyDesc(nat.MODEL_3DGS, float(cfg.grad_threshold), float(cfg.split_scale),
                               float(cfg.min_opacity), float(cfg.max_scale), int(cfg.seed) & 0xFFFFFFFF)
        action = torch.empty(max(S, 1), dtype=torch.int32, device=dev)
        gout = torch.zeros(max(ng, 1), dtype=torch.int32, device=dev)
        stats = self.densify_stats if self.densify_stats is not None and self.densify_stats.shape[0] >= S else None
        nat.call("bs_densify_mark", desc, nat.ptr(self.params), S, nat.ptr(stats), nat.ptr(self.group_begin), ng,
                 nat.ptr(action), nat.ptr(gout), st)
        new_begin = torch.zeros(ng + 1, dtype=torch.int32, device=dev)
        new_begin[1:] = torch.cumsum(gout[:ng], 0, dtype=torch.int32)
        S_new = int(new_begin[-1].item())
        params = torch.empty(nat.PARAM_PLANES, max(S_new, 1), 4, dtype=torch.float32, device=dev)
        m = torch.empty_like(params)
        v = torch.empty_like(params)
        src = torch.empty(max(S_new, 1), dtype=torch.int32, device=dev)
        nat.call("bs_densify_apply", desc, nat.ptr(self.params), nat.ptr(self.exp_avg), nat.ptr(self.exp_avg_sq), S,
                 nat.ptr(action), nat.ptr(self.group_begin), nat.ptr(new_begin), ng, nat.ptr(self.global_ids),
                 nat.ptr(params), nat.ptr(m), nat.ptr(v), S_new, nat.ptr(src), st)
        aabb = torch.empty(max(ng, 1), 6, dtype=torch.float32, device=dev)
        nat.call("bs_group_aabb_ranges", nat.ptr(params), S_new, nat.ptr(new_begin), ng, nat.ptr(aabb), st)
        counts = torch.bincount(action[:S].long(), minlength=4).cpu().numpy()
        sizes = np.diff(new_begin.cpu().numpy().astype(np.int64))
        # the new shard
        self.params, self.exp_avg, self.exp_avg_sq = params[:, :S_new], m[:, :S_new], v[:, :S_new]
        self.S = S_new
        self.group_begin = new_begin
        self.aabb = aabb[:ng]
        self.max_group = int(sizes.max()) if len(sizes) else 0
        self.max_chunks = max(1, -(-self.max_group // 256))
        if self.presence is not None:
            self.presence = self.presence.index_select(0, src[:S_new].long())
        if self.comm is not None or self.global_ids is not None:
            self.global_ids = torch.as_tensor(self._renumber(sizes), device=dev)
        if self.densify_stats is not None:
            self.densify_stats = torch.zeros(max(S_new, 1), 2, dtype=torch.float32, device=dev)
        self.last = {}
        return {"n_before": int(S), "n_after": int(S_new), "pruned": int(counts[nat.DENSIFY_PRUNE]),
                "kept": int(counts[nat.DENSIFY_KEEP]), "cloned": int(counts[nat.DENSIFY_CLONE]),
                "split": int(counts[nat.DENSIFY_SPLIT]), "src_index": src[:S_new]}

    def _renumber(self, sizes: np.ndarray) -> np.ndarray:
        """Global ids after densification: groups of all ranks in global key
        order, points consecutively inside each group (the single-rank
        numbering for any number of ranks)."""
        keys, sizes = np.asarray(self.group_keys, dtype=np.int64), np.asarray(sizes, dtype=np.int64)
        if self.comm is not None:
            import torch.distributed as dist

            grp = getattr(self.comm, "group", None)
            parts = [None] * dist.get_world_size(grp)
            dist.all_gather_object(parts, (keys.tolist(), sizes.tolist()), group=grp)
            all_keys = np.concatenate([np.asarray(k, dtype=np.int64) for k, _ in parts])
            all_sizes = np.concatenate([np.asarray(z, dtype=np.int64) for _, z in parts])
        else:
            all_keys, all_sizes = keys, sizes
        order = np.argsort(all_keys, kind="stable")
        start = np.zeros(len(all_keys), dtype=np.int64)
        start[order] = np.concatenate([[0], np.cumsum(all_sizes[order])[:-1]]) if len(order) else []
        lut = dict(zip(all_keys.tolist(), start.tolist()))
        ids = np.concatenate([lut[int(k)] + np.arange(n, dtype=np.int64) for k, n in zip(keys, sizes)]) \
            if len(keys) else np.zeros(0, dtype=np.int64)
        if len(ids) and ids[-1] >= 2**31:
            raise ValueError("global ids exceed int32 after densification")
        return ids.astype(np.int32)

    # ------------------------------------------------------------------ checkpoint
    def state_dict(self) -> dict:
        """The rank's training state (shard parameters, Adam moments, step
        counter; SURVEY.md §5 checkpoint/resume): `torch.save` it per rank.
        It carries the shard layout too (group table, AABBs, global ids,
        densification statistic), which densification changes."""
        sd = {"params": self.params.detach().clone(), "exp_avg": self.exp_avg.detach().clone(),
              "exp_avg_sq": self.exp_avg_sq.detach().clone(), "step": int(self.step_count),
              "model": self.model, "n_points": int(self.S),
              "group_begin": self.group_begin.detach().clone(), "aabb": self.aabb.detach().clone(),
              "group_keys": torch.as_tensor(np.asarray(self.group_keys, dtype=np.int64))}
        for name in ("global_ids", "presence", "densify_stats"):
            t = getattr(self, name)
            sd[name] = None if t is None else t.detach().clone()
        return sd

    def load_state_dict(self, sd: dict) -> None:
        """Resume from state_dict(); a checkpoint taken after densification
        (another point count, same groups) replaces the shard layout."""
        from .status import ConsistencyError

        n = int(sd.get("n_points", -1))
        if sd.get("model") != self.model:
            raise ConsistencyError("checkpoint is of a different model")
        if n != self.S and ("group_begin" not in sd or len(sd["group_begin"]) != self.n_groups + 1):
            raise ConsistencyError("checkpoint is of a different shard")
        if n != self.S:
            for name in ("params", "exp_avg", "exp_avg_sq"):
                setattr(self, name, sd[name].to(self.dev).clone())
        else:
            for name in ("params", "exp_avg", "exp_avg_sq"):
                getattr(self, name).copy_(sd[name].to(self.dev))
        if "group_begin" in sd:
            self.S = n
            self.group_begin = sd["group_begin"].to(self.dev).clone()
            self.aabb = sd["aabb"].to(self.dev).clone()
            self.group_keys = np.asarray(sd["group_keys"].cpu().numpy(), dtype=np.int64)
            sizes = np.diff(self.group_begin.cpu().numpy().astype(np.int64))
            self.max_group = int(sizes.max()) if len(sizes) else 0
            self.max_chunks = max(1, -(-self.max_group // 256))
            for name in ("global_ids", "presence", "densify_stats"):
                t = sd.get(name)
                setattr(self, name, None if t is None else t.to(self.dev).clone())
        self.step_count = int(sd["step"])
        self.last = {}

    def _single_pass_bin(self, pdesc, B, n_rows):
        """Zeroed (view, tile) bucket counters and the per-row tile records the
        projection fills (bs_proj_desc.bucket_counts / row_bin)."""
        counts_b = self.buf.get("bucket_counts", B * self.tiles, torch.int32)
        counts_b.zero_()
        records = self.buf.get("row_bin", max(n_rows, 1) * 4, torch.int32)
        pdesc.bucket_counts, pdesc.row_bin, pdesc.tiles_per_slot = nat.ptr(counts_b), nat.ptr(records), self.tiles
        return records

    def _canonical(self, sp_recv, gid_recv, n, seg_rows, seg_slot, n_slots):
        """Received rows -> canonical order (slot-major, ascending global id;
        bs_canonical_order).  Returns the reordered rows and `order`
        (canonical position -> received row)."""
        st, lib = nat.stream_handle(), nat.load()
        seg_row0 = self._up(np.concatenate([[0], np.cumsum(seg_rows)[:-1]]), "canon_seg_row0", torch.int64)
        seg_slot_t = self._up(seg_slot, "canon_seg_slot", torch.int32)
        order = self.buf.get("canon_order", max(n, 1), torch.int64)
        cgid = self.buf.get("canon_gid", max(n, 1), torch.int32)
        ws = self.buf.get("canon_ws", lib.bs_canonical_order_workspace(max(n, 1)), torch.uint8)
        nat.call("bs_canonical_order", nat.ptr(gid_recv), n, nat.ptr(seg_row0), nat.ptr(seg_slot_t), len(seg_slot),
                 n_slots, nat.ptr(order), nat.ptr(cgid), nat.ptr(ws), ws.numel(), st)
        sp_c = self.buf.get("sp_canon", max(n, 1) * self.sp_floats, torch.float32)
        nat.call("bs_gather_rows", nat.ptr(sp_recv), self.sp_floats, nat.ptr(order), n, nat.ptr(sp_c), st)
        sup = self.buf.get("row_support", max(n, 1), torch.float32)
        nat.call("bs_row_support", nat.ptr(sp_c), self.model_id, n, nat.ptr(sup), st)
        self.last["row_gid"] = cgid[:n]
        self._recv_support = sup
        return sp_c, order

    def _uncanonical(self, gsp_c, order, n, wire):
        """G_SP rows of the canonical order -> received order, `wire` floats each."""
        g = self.buf.get("gsp_wire", max(n, 1) * wire, torch.float32)[: n * wire]
        g.zero_()
        nat.call("bs_scatter_add_rows", nat.ptr(gsp_c), self.gsp_floats, wire, nat.ptr(order), n, nat.ptr(g), wire,
                 nat.stream_handle())
        return g

    def _adam_desc(self):
        ad = nat.AdamDesc()
        for k in range(60):
            ad.lr[k] = float(self.adam.lr[k])
        ad.beta1, ad.beta2, ad.eps = self.adam.beta1, self.adam.beta2, self.adam.eps
        ad.step, ad.selective = self.step_count, 1 if self.adam.selective else 0
        return ad

    def _slot_ids(self, B):
        t = self.buf.bufs.get("slot_ids")
        if t is None or t.numel() < 32:
            t = torch.arange(32, dtype=torch.int32, device=self.dev)
            self.buf.bufs["slot_ids"] = t
        return t[:B]

    def _bin_buckets(self, sp, n_rows, seg_row0, seg_slot, n_slots, slot_cams, before_sync=None, records=None):
        """Bucket pipeline (csrc/bin_tiles.cu), see binning.bin_buckets."""
        n_inst, irows, ranges, biggest = bin_buckets(self.buf, sp, n_rows, seg_row0, seg_slot, n_slots, slot_cams,
                                                     self.tiles, self.model_id, self.sort_cap, before_sync,
                                                     self.bin_capacity_hint, records=records)
        self.last["largest_bucket"] = biggest
        return n_inst, irows, ranges

    def _bin_radix(self, sp, n_rows, seg_row0, seg_slot, n_slots, slot_cams):
        """Radix pipeline (csrc/bin.cu + sort.cu): stable depth sort of the rows,
        tile emission in depth order, stable tile sort, ranges."""
        st, lib = nat.stream_handle(), nat.load()
        keys = self.buf.get("dkeys", max(n_rows, 1), torch.int64)
        vals = self.buf.get("dvals", max(n_rows, 1), torch.int32)
        nat.call("bs_bin_depth_keys", nat.ptr(sp), n_rows, nat.ptr(seg_row0), nat.ptr(seg_slot),
                 len(seg_slot), nat.ptr(keys), nat.ptr(vals), st)
        ka = self.buf.get("dkeys_alt", max(n_rows, 1), torch.int64)
        va = self.buf.get("dvals_alt", max(n_rows, 1), torch.int32)
        ws = self.buf.get("sort_ws", lib.bs_radix_sort_workspace(max(n_rows, 1)), torch.uint8)
        nat.call("bs_radix_sort_u64", nat.ptr(keys), nat.ptr(vals), nat.ptr(ka), nat.ptr(va), n_rows, None, 0,
                 32 + _bits_for(n_slots), nat.ptr(ws), ws.numel(), st)
        offsets = self.buf.get("offsets", max(n_rows, 1), torch.int64)
        total = self.buf.get("total", 1, torch.int64)
        cws = self.buf.get("count_ws", lib.bs_bin_count_workspace(max(n_rows, 1)), torch.uint8)
        nat.call("bs_bin_count", nat.ptr(sp), nat.ptr(vals), n_rows, nat.ptr(keys), nat.ptr(slot_cams),
                 nat.ptr(offsets), nat.ptr(total), nat.ptr(cws), cws.numel(), st)
        n_inst = int(total.item())  # sync 2: sizes the instance buffers
        ikeys = self.buf.get("ikeys", max(n_inst, 1), torch.int32)
        irows = self.buf.get("irows", max(n_inst, 1), torch.int32)
        nat.call("bs_bin_emit", nat.ptr(sp), nat.ptr(vals), n_rows, nat.ptr(keys), nat.ptr(slot_cams),
                 self.tiles, nat.ptr(offsets), nat.ptr(ikeys), nat.ptr(irows), st)
        ika = self.buf.get("ikeys_alt", max(n_inst, 1), torch.int32)
        ira = self.buf.get("irows_alt", max(n_inst, 1), torch.int32)
        ws2 = self.buf.get("sort_ws2", lib.bs_radix_sort_workspace(max(n_inst, 1)), torch.uint8)
        nat.call("bs_radix_sort_u32", nat.ptr(ikeys), nat.ptr(irows), nat.ptr(ika), nat.ptr(ira), n_inst, None,
                 0, _bits_for(n_slots * self.tiles), nat.ptr(ws2), ws2.numel(), st)
        ranges = self.buf.get("ranges", n_slots * self.tiles * 2, torch.int32)
        nat.call("bs_tile_ranges", nat.ptr(ikeys), None, n_inst, n_slots * self.tiles, nat.ptr(ranges), st)
        return n_inst, irows, ranges

    def _render_and_backward(self, sp, n_rows, seg_row0, seg_slot, n_slots, slot_cams, gt_views, gt_batch,
                             slot_patches=None, gsp_cleared=False, support=None, records=None):
        dev, st = self.dev, nat.stream_handle()
        lib = nat.load()
        gsp = self.buf.get("gsp", max(n_rows, 1) * self.gsp_floats, torch.float32)
        # ---- K2: binning
        with self._t("bin"):
            if self.binning == "radix":
                if self.model != "3dgs":
                    raise ValueError("the radix binning pipeline reads 3DGS rows only; use binning='bucket'")
                gsp.zero_()
                n_inst, irows, ranges = self._bin_radix(sp, n_rows, seg_row0, seg_slot, n_slots, slot_cams)
            else:
                # the G_SP accumulator is cleared while the host reads the instance count
                n_inst, irows, ranges = self._bin_buckets(sp, n_rows, seg_row0, seg_slot, n_slots, slot_cams,
                                                          before_sync=None if gsp_cleared else gsp.zero_,
                                                          records=records)
        self.last.update(n_rows=n_rows, n_inst=n_inst, n_slots=n_slots)
        # ---- K3: forward + fused L1 partials
        npx = self.H * self.W
        image = self.buf.get("image", n_slots * npx * 3, torch.float32)
        final_T = self.buf.get("final_T", n_slots * npx, torch.float32)
        n_contrib = self.buf.get("n_contrib", n_slots * npx, torch.int32)
        loss_tiles = self.buf.get("loss_tiles", n_slots * self.tiles, torch.float32)
        rdesc = nat.RasterDesc(n_slots, self.tiles, self.W, self.H, (ctypes.c_float * 3)(*self.bg), 1,
                               self.pixels_per_lane, self.P, nat.ptr(slot_patches), nat.ptr(support))
        if gt_batch is not None:
            self._wait_gt()
            gt, gt_map = gt_batch, None
        else:
            gt = self.gt
            gt_map = self._select_views(gt_views, self._gt_index, "gt_map")  # host view ids -> gt rows
        losses = self.buf.get("losses", n_slots, torch.float32)
        if self.raster_fused and (self.model == "2dgs" or self.pixels_per_lane == 1):
            # K3 + L + K4 in one launch: each warp keeps its forward's splat list in shared memory
            with self._t("raster"):
                aux = self.keep_raster_aux
                nat.call("bs_raster2d_fwd_bwd" if self.model == "2dgs" else "bs_raster_fwd_bwd", rdesc, nat.ptr(sp),
                         nat.ptr(irows), nat.ptr(ranges), nat.ptr(image), nat.ptr(final_T) if aux else None,
                         nat.ptr(n_contrib) if aux else None, nat.ptr(gt), nat.ptr(gt_map), nat.ptr(loss_tiles),
                         nat.ptr(gsp), st)
            nat.call("bs_reduce_loss_tiles", nat.ptr(loss_tiles), n_slots, self.tiles, self.H, self.W,
                     nat.ptr(losses), st)
        else:
            with self._t("raster_fwd"):
                nat.call(self._raster[0], rdesc, nat.ptr(sp), nat.ptr(irows), nat.ptr(ranges), nat.ptr(image),
                         nat.ptr(final_T), nat.ptr(n_contrib), nat.ptr(gt), nat.ptr(gt_map), nat.ptr(loss_tiles), st)
            nat.call("bs_reduce_loss_tiles", nat.ptr(loss_tiles), n_slots, self.tiles, self.H, self.W,
                     nat.ptr(losses), st)
            # ---- K4: backward
            with self._t("raster_bwd"):
                nat.call(self._raster[1], rdesc, nat.ptr(sp), nat.ptr(irows), nat.ptr(ranges), nat.ptr(image),
                         nat.ptr(final_T), nat.ptr(n_contrib), None, nat.ptr(gt), nat.ptr(gt_map), nat.ptr(gsp), st)
        self.last.update(image=image, final_T=final_T, n_contrib=n_contrib, ranges=ranges, irows=irows,
                         sp=sp, gsp=gsp)
        return losses, gsp
