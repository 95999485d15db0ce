"""Z-order grouping, frusta, culling and the access matrix A.

API shape of /root/reference/pkg/src/splatsched/visibility.py (morton_codes,
zorder_group, Frustum, frustum_from_view, patch_frusta, cull_points,
cull_group, build_access_matrix); the per-point work runs in the sm_100a
kernel K0 (``bs_cull_count``) and the Morton/radix-sort kernels.  Frustum
planes are built on the host with the same numpy operations as the reference
(visibility.py:168-217) and uploaded as float64, so point/patch membership
is bit-exact with the reference (see csrc/cull.cu for the evaluation order).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .scenes import CameraView, PointCloud
from .status import ConfigurationError, ConsistencyError, ParameterError

OUTSIDE = "outside"
INTERSECTING = "intersecting"
EXACT = "exact"
GROUP_APPROX = "group_approx"
DEFAULT_GROUP_SIZE = 2048
DEFAULT_BITS_PER_AXIS = 21


# ---------------------------------------------------------------------------
# frusta (host, float64)


def _unit(v: np.ndarray) -> np.ndarray:
    return v / np.linalg.norm(v)


def _x_edge(view: CameraView, px) -> np.ndarray:
    slope = (2.0 * px / view.width - 1.0) * math.tan(view.fov_x / 2.0)
    return _unit(np.array([1.0, 0.0, -slope]))


def _y_edge(view: CameraView, py) -> np.ndarray:
    slope = (2.0 * py / view.height - 1.0) * math.tan(view.fov_y / 2.0)
    return _unit(np.array([0.0, 1.0, -slope]))


def _world_plane(view: CameraView, n_cam: np.ndarray, c_cam: float) -> np.ndarray:
    n = view.rotation @ n_cam
    out = np.empty(4)
    out[:3] = n
    out[3] = c_cam - n @ view.position
    return out


def patch_edges(extent: int, P: int) -> list[int]:
    return [(c * extent) // P for c in range(P)] + [extent]


@dataclass
class Frustum:
    """Six (normal, offset) planes: near, far, left, right(excl), top, bottom(excl)."""

    planes: np.ndarray
    inclusive: np.ndarray

    def signed_distances(self, positions) -> np.ndarray:
        p = np.atleast_2d(positions).astype(np.float64)
        return p @ self.planes[:, :3].T + self.planes[:, 3]

    def contains(self, positions) -> np.ndarray:
        d = self.signed_distances(positions)
        return np.where(self.inclusive, d >= 0.0, d > 0.0).all(axis=1)


def frustum_from_view(view: CameraView, patch=None) -> Frustum:
    """Frustum of a view restricted to the half-open pixel rectangle `patch`."""
    x0, y0, x1, y1 = (0, 0, view.width, view.height) if patch is None else patch
    if not (0 <= x0 < x1 <= view.width and 0 <= y0 < y1 <= view.height):
        raise ParameterError(f"patch rectangle {patch} invalid for {view.width}x{view.height} image")
    rows = [
        (np.array([0.0, 0.0, 1.0]), -view.near),
        (np.array([0.0, 0.0, -1.0]), view.far),
        (_x_edge(view, x0), 0.0),
        (-_x_edge(view, x1), 0.0),
        (_y_edge(view, y0), 0.0),
        (-_y_edge(view, y1), 0.0),
    ]
    planes = np.stack([_world_plane(view, n, c) for n, c in rows])
    return Frustum(planes, np.array([True, True, True, False, True, False]))


def patch_frusta(view: CameraView, P: int) -> list[Frustum]:
    if P < 1:
        raise ParameterError("patch factor P must be >= 1")
    xs, ys = patch_edges(view.width, P), patch_edges(view.height, P)
    return [frustum_from_view(view, (xs[c], ys[r], xs[c + 1], ys[r + 1])) for r in range(P) for c in range(P)]


def view_plane_block(view: CameraView, P: int) -> np.ndarray:
    """float64 [2 + 2(P+1), 4]: near, far, x-edge planes c=0..P, y-edge planes
    r=0..P -- the shared planes of all P*P patch frusta of `view`
    (bs_cull_count layout)."""
    if P < 1:
        raise ParameterError("patch factor P must be >= 1")
    xs, ys = patch_edges(view.width, P), patch_edges(view.height, P)
    rows = [_world_plane(view, np.array([0.0, 0.0, 1.0]), -view.near),
            _world_plane(view, np.array([0.0, 0.0, -1.0]), view.far)]
    rows += [_world_plane(view, _x_edge(view, x), 0.0) for x in xs]
    rows += [_world_plane(view, _y_edge(view, y), 0.0) for y in ys]
    return np.stack(rows)


def batch_planes(views, P: int) -> np.ndarray:
    return np.ascontiguousarray(np.stack([view_plane_block(v, P) for v in views]))


def cull_points(frustum: Frustum, positions, view_time=None, presence=None) -> np.ndarray:
    """Host-side visibility mask (API compatibility; the hot path is K0)."""
    if (view_time is None) != (presence is None):
        raise ConfigurationError("view_time and presence intervals must be supplied together")
    mask = frustum.contains(positions)
    if view_time is not None:
        pres = np.atleast_2d(presence)
        mask &= (pres[:, 0] <= view_time) & (view_time <= pres[:, 1])
    return mask


def cull_point(frustum, point, view_time=None, presence=None) -> bool:
    p = np.asarray(point.as_array() if hasattr(point, "as_array") else point, dtype=np.float64).reshape(1, 3)
    pres = None if presence is None else np.asarray(presence).reshape(1, 2)
    return bool(cull_points(frustum, p, view_time, pres)[0])


def cull_group(frustum: Frustum, aabb) -> str:
    box = np.asarray(aabb, dtype=np.float64)
    if (box[0] > box[1]).any():
        raise ParameterError("AABB must have min <= max per axis")
    corners = np.array([[box[i, 0], box[j, 1], box[k, 2]] for i in (0, 1) for j in (0, 1) for k in (0, 1)])
    return OUTSIDE if (frustum.signed_distances(corners) < 0.0).all(axis=0).any() else INTERSECTING


# ---------------------------------------------------------------------------
# Morton codes and grouping (GPU)


def _dev():
    nat.load()
    return torch.device("cuda", torch.cuda.current_device())


def morton_codes(positions, bbox, bits_per_axis: int = DEFAULT_BITS_PER_AXIS) -> np.ndarray:
    if not (1 <= bits_per_axis <= 21):
        raise ParameterError("bits_per_axis must be in [1, 21]")
    dev = _dev()
    pos = torch.as_tensor(np.ascontiguousarray(np.atleast_2d(positions), dtype=np.float32), device=dev)
    bb = torch.as_tensor(np.asarray(bbox, dtype=np.float32).reshape(6), device=dev)
    codes = torch.empty(len(pos), dtype=torch.int64, device=dev)
    nat.call("bs_morton_codes", nat.ptr(pos), len(pos), 3, nat.ptr(bb), bits_per_axis, nat.ptr(codes),
             nat.stream_handle())
    return codes.cpu().numpy().view(np.uint64)


def morton_code(point, bbox, bits_per_axis: int = DEFAULT_BITS_PER_AXIS) -> int:
    p = np.asarray(point.as_array() if hasattr(point, "as_array") else point, dtype=np.float64)
    return int(morton_codes(p.reshape(1, 3), bbox, bits_per_axis)[0])


def radix_sort_u64(keys: torch.Tensor, vals: torch.Tensor, begin_bit: int = 0, end_bit: int = 64):
    """Stable sort of (u64 key stored as int64, u32 value stored as int32) pairs, in place."""
    n = keys.numel()
    ka = torch.empty_like(keys)
    va = torch.empty_like(vals)
    ws = torch.empty(nat.load().bs_radix_sort_workspace(n), dtype=torch.uint8, device=keys.device)
    nat.call("bs_radix_sort_u64", nat.ptr(keys), nat.ptr(vals), nat.ptr(ka), nat.ptr(va), n, None, begin_bit,
             end_bit, nat.ptr(ws), ws.numel(), nat.stream_handle())
    return keys, vals


@dataclass(frozen=True)
class PointGroup:
    group_id: int
    begin: int
    end: int
    aabb: np.ndarray

    @property
    def size(self) -> int:
        return self.end - self.begin


@dataclass
class GroupedCloud:
    """Z-order-sorted cloud in groups of at most G points;
    sorted_cloud[i] == original_cloud[permutation[i]]."""

    sorted_cloud: PointCloud
    permutation: np.ndarray
    groups: list
    group_size: int
    aabbs: np.ndarray = None  # (n_groups, 2, 3) float32
    _device: dict = field(default_factory=dict, repr=False)

    @property
    def n_groups(self) -> int:
        return len(self.groups)

    def group_of_point(self) -> np.ndarray:
        return np.repeat(np.arange(self.n_groups, dtype=np.int64),
                         [g.size for g in self.groups]) if self.groups else np.empty(0, np.int64)

    def group_begin(self) -> np.ndarray:
        return np.array([g.begin for g in self.groups] + [len(self.sorted_cloud)], dtype=np.int32)

    def device_arrays(self, dev):
        """(positions f32 [n,3], group_begin i32, aabb f32 [ng,6], presence) on `dev`, cached."""
        key = str(dev)
        if key not in self._device:
            pres = self.sorted_cloud.timestamps
            self._device[key] = (
                torch.as_tensor(self.sorted_cloud.positions, device=dev).contiguous(),
                torch.as_tensor(self.group_begin(), device=dev),
                torch.as_tensor(np.ascontiguousarray(self.aabbs.reshape(-1, 6)), device=dev),
                None if pres is None else torch.as_tensor(pres, device=dev).contiguous(),
            )
        return self._device[key]


def zorder_group(cloud: PointCloud, G: int = DEFAULT_GROUP_SIZE,
                 bits_per_axis: int = DEFAULT_BITS_PER_AXIS) -> GroupedCloud:
    """Stable Morton sort (GPU radix sort) + groups of G with AABBs."""
    if G < 1:
        raise ParameterError("group size G must be >= 1")
    if not (1 <= bits_per_axis <= 21):
        raise ParameterError("bits_per_axis must be in [1, 21]")
    dev = _dev()
    n = len(cloud)
    st = nat.stream_handle()
    pos = torch.as_tensor(cloud.positions, device=dev).contiguous()
    bbox = torch.empty(6, dtype=torch.float32, device=dev)
    ws = torch.empty(nat.load().bs_bbox_workspace(n), dtype=torch.uint8, device=dev)
    nat.call("bs_bbox", nat.ptr(pos), n, 3, nat.ptr(bbox), nat.ptr(ws), ws.numel(), st)
    codes = torch.empty(n, dtype=torch.int64, device=dev)
    nat.call("bs_morton_codes", nat.ptr(pos), n, 3, nat.ptr(bbox), bits_per_axis, nat.ptr(codes), st)
    perm = torch.arange(n, dtype=torch.int32, device=dev)
    radix_sort_u64(codes, perm, 0, 3 * bits_per_axis)
    perm64 = perm.to(torch.int64)
    spos = torch.empty_like(pos)
    # gather rows of 3 floats: treat as 1 plane of float4? rows are 12 B, use torch index (plumbing)
    spos.copy_(pos.index_select(0, perm64))
    ng = (n + G - 1) // G
    aabb = torch.empty(ng * 6, dtype=torch.float32, device=dev)
    nat.call("bs_group_aabb", nat.ptr(spos), n, 3, G, nat.ptr(aabb), st)
    perm_np = perm64.cpu().numpy()
    aabb_np = aabb.cpu().numpy().reshape(ng, 2, 3)
    sorted_cloud = PointCloud(cloud.positions[perm_np], None if cloud.timestamps is None
                              else cloud.timestamps[perm_np])
    groups = [PointGroup(g, g * G, min(g * G + G, n), aabb_np[g]) for g in range(ng)]
    gc = GroupedCloud(sorted_cloud, perm_np, groups, G, aabb_np)
    pres = sorted_cloud.timestamps
    gc._device[str(dev)] = (spos, torch.as_tensor(gc.group_begin(), device=dev), aabb,
                            None if pres is None else torch.as_tensor(pres, device=dev))
    return gc


# ---------------------------------------------------------------------------
# access matrix (GPU K0)


def point_gpu_from_partition(grouped: GroupedCloud, partition) -> np.ndarray:
    if partition.n_groups != grouped.n_groups:
        raise ConsistencyError(f"partition covers {partition.n_groups} groups, cloud has {grouped.n_groups}")
    return np.repeat(partition.flat_gpus().astype(np.int64), [g.size for g in grouped.groups])


def build_access_matrix(grouped: GroupedCloud, partition, batch, P: int = 1, granularity: str = EXACT,
                        temporal: bool = False) -> np.ndarray:
    """(B*P*P, N) int64 counts of in-frustum points per patch and GPU
    (row = view_pos * P^2 + patch_row * P + patch_col), computed by K0."""
    if isinstance(partition, np.ndarray):
        point_gpu = partition.astype(np.int64)
        if len(point_gpu) != len(grouped.sorted_cloud):
            raise ConsistencyError("per-point GPU array length mismatch")
        n_gpus = int(point_gpu.max()) + 1 if len(point_gpu) else 1
    else:
        point_gpu = point_gpu_from_partition(grouped, partition)
        n_gpus = partition.n_gpus
    if granularity not in (EXACT, GROUP_APPROX):
        raise ParameterError(f"unknown granularity {granularity!r}")
    if P < 1:
        raise ParameterError("patch factor P must be >= 1")
    if temporal and grouped.sorted_cloud.timestamps is None:
        raise ConfigurationError("temporal culling requested without timestamps")
    batch = list(batch)
    if temporal:
        for v in batch:
            if v.time is None:
                raise ConfigurationError(f"view {v.id} lacks a timestamp")
    dev = _dev()
    pos, gbeg, aabb, pres = grouped.device_arrays(dev)
    gpu = torch.as_tensor(point_gpu.astype(np.int32), device=dev)
    out_rows = []
    # chunk views so the per-CTA plane table stays within shared memory
    chunk = max(1, min(len(batch), 4096 // (2 + 2 * (P + 1))))
    for s in range(0, len(batch), chunk):
        views = batch[s:s + chunk]
        planes = torch.as_tensor(batch_planes(views, P), device=dev)
        vt = torch.as_tensor(np.array([v.time for v in views], dtype=np.float32), device=dev) if temporal else None
        out = torch.empty((len(views) * P * P, n_gpus), dtype=torch.int64, device=dev)
        desc = nat.CullDesc(nat.CULL_ACCESS_EXACT if granularity == EXACT else nat.CULL_ACCESS_GROUP,
                            len(views), P, n_gpus, 1 if temporal else 0, 3)
        nat.call("bs_cull_count", desc, nat.ptr(pos), len(pos), nat.ptr(pres) if temporal else None, nat.ptr(gbeg),
                 nat.ptr(aabb), grouped.n_groups, nat.ptr(planes), nat.ptr(vt), nat.ptr(gpu), nat.ptr(out), None,
                 None, nat.stream_handle())
        out_rows.append(out)
    return torch.cat(out_rows).cpu().numpy()
