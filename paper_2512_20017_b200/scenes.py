"""Point/camera data model and synthetic scene inputs.

Shapes and validation mirror the reference's data model
(/root/reference/pkg/src/splatsched/scene.py:27-205) so code written against
``splatsched`` keeps working: ``PointCloud`` (f32 positions, optional f32
presence intervals), ``CameraView`` (pinhole, +x right / +y down / +z
forward, ``rotation`` camera->world), ``WorkloadProfile`` and
``SceneDataset``.  The two generators reproduce the reference's RNG streams
call-for-call (scene.py:212-215, 282-462), so positions and cameras are
bit-identical to ``splatsched.generate_*_scene`` for the same arguments --
the parity tests rely on that.

New here: ``GaussianModel`` -- the trainable 3DGS state (59 floats per
point) laid out in the plane-major float4 format of the
kernels (include/splat_b200.h), initialised from an independent RNG stream
``SeedSequence([seed, 4])``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .status import ParameterError

CULLING_SPATIAL = "spatial"
CULLING_SPATIOTEMPORAL = "spatiotemporal"


@dataclass(frozen=True)
class WorkloadProfile:
    """View-dependent splat-state size of one workload (elements x bytes)."""

    name: str
    splat_state_elements: int
    bytes_per_element: int = 4
    culling_mode: str = CULLING_SPATIAL

    def __post_init__(self):
        if self.splat_state_elements <= 0 or self.bytes_per_element <= 0:
            raise ParameterError("profile sizes must be positive")
        if self.culling_mode not in (CULLING_SPATIAL, CULLING_SPATIOTEMPORAL):
            raise ParameterError(f"unknown culling_mode {self.culling_mode!r}")

    @property
    def bytes_per_point(self) -> int:
        return self.splat_state_elements * self.bytes_per_element

    @property
    def temporal(self) -> bool:
        return self.culling_mode == CULLING_SPATIOTEMPORAL


PROFILE_3DGS = WorkloadProfile("3dgs", 11)
PROFILE_2DGS = WorkloadProfile("2dgs", 20)
PROFILE_3DCX = WorkloadProfile("3dcx", 29)
PROFILE_4DGS = WorkloadProfile("4dgs", 11, culling_mode=CULLING_SPATIOTEMPORAL)
BUILTIN_PROFILES = {p.name: p for p in (PROFILE_3DGS, PROFILE_2DGS, PROFILE_3DCX, PROFILE_4DGS)}


@dataclass(frozen=True)
class Point3:
    x: float
    y: float
    z: float

    def __post_init__(self):
        if not all(math.isfinite(v) for v in (self.x, self.y, self.z)):
            raise ParameterError("point coordinates must be finite")

    def as_array(self) -> np.ndarray:
        return np.array([self.x, self.y, self.z], dtype=np.float64)


class PointCloud:
    """Positions (n, 3) float32 and optional presence intervals (n, 2) float32."""

    def __init__(self, positions, timestamps=None):
        pos = np.asarray(positions, dtype=np.float32)
        if pos.ndim != 2 or pos.shape[1] != 3:
            raise ParameterError("positions must have shape (n, 3)")
        if len(pos) == 0:
            raise ParameterError("point cloud must be non-empty")
        if not np.isfinite(pos).all():
            raise ParameterError("positions must be finite")
        self.positions = pos
        self.timestamps = None
        if timestamps is not None:
            ts = np.asarray(timestamps, dtype=np.float32)
            if ts.shape != (len(pos), 2):
                raise ParameterError("timestamps must have shape (n, 2)")
            if (ts[:, 0] > ts[:, 1]).any():
                raise ParameterError("presence intervals need t_start <= t_end")
            self.timestamps = ts

    def __len__(self) -> int:
        return len(self.positions)

    @property
    def bbox(self) -> np.ndarray:
        return np.stack([self.positions.min(axis=0), self.positions.max(axis=0)])

    def __eq__(self, other):
        if not isinstance(other, PointCloud):
            return NotImplemented
        if not np.array_equal(self.positions, other.positions):
            return False
        if (self.timestamps is None) != (other.timestamps is None):
            return False
        return self.timestamps is None or np.array_equal(self.timestamps, other.timestamps)


class CameraView:
    """Pinhole camera; ``rotation`` maps camera-frame vectors to world."""

    def __init__(self, id, position, rotation, fov_x, fov_y, near, far, width, height, time=None):
        self.id = id
        self.position = np.asarray(position, dtype=np.float64)
        self.rotation = np.asarray(rotation, dtype=np.float64)
        self.fov_x, self.fov_y = fov_x, fov_y
        self.near, self.far = near, far
        self.width, self.height = width, height
        self.time = time
        if self.position.shape != (3,) or self.rotation.shape != (3, 3):
            raise ParameterError("camera position must be (3,) and rotation (3, 3)")
        if not (0 < near < far):
            raise ParameterError("camera needs 0 < near < far")
        if not (0 < fov_x < math.pi and 0 < fov_y < math.pi):
            raise ParameterError("fov must be in (0, pi)")
        if width < 1 or height < 1:
            raise ParameterError("image size must be >= 1 pixel")
        err = np.abs(self.rotation @ self.rotation.T - np.eye(3)).max()
        if err > 1e-9:
            raise ParameterError(f"rotation not orthonormal (error {err:g})")

    @property
    def forward(self) -> np.ndarray:
        return self.rotation[:, 2]

    def intrinsics(self):
        """(fx, fy, cx, cy) of the test_visibility.py:204-215 convention."""
        tx, ty = math.tan(self.fov_x / 2.0), math.tan(self.fov_y / 2.0)
        return self.width / (2.0 * tx), self.height / (2.0 * ty), self.width / 2.0, self.height / 2.0

    def __eq__(self, other):
        if not isinstance(other, CameraView):
            return NotImplemented
        return (self.id == other.id and np.array_equal(self.position, other.position)
                and np.array_equal(self.rotation, other.rotation)
                and (self.fov_x, self.fov_y, self.near, self.far, self.width, self.height, self.time)
                == (other.fov_x, other.fov_y, other.near, other.far, other.width, other.height, other.time))

    def __repr__(self):
        return f"CameraView(id={self.id}, {self.width}x{self.height})"


class SceneDataset:
    def __init__(self, cloud: PointCloud, views, profile: WorkloadProfile):
        self.cloud, self.views, self.profile = cloud, list(views), profile
        if [v.id for v in self.views] != list(range(len(self.views))):
            raise ParameterError("view ids must be unique and contiguous from 0")
        if profile.temporal and (cloud.timestamps is None or any(v.time is None for v in self.views)):
            raise ParameterError("spatio-temporal profile requires point and view timestamps")

    def __eq__(self, other):
        if not isinstance(other, SceneDataset):
            return NotImplemented
        return self.cloud == other.cloud and self.views == other.views and self.profile == other.profile


# ---------------------------------------------------------------------------
# generators (RNG streams of scene.py:212-219, 282-462)


def _stream(seed: int, k: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed), k]))


def _arclength_resample(points: np.ndarray, n: int) -> np.ndarray:
    """n positions evenly spaced by arclength along a polyline."""
    if n == 1:
        return points[:1].copy()
    seg = np.diff(points, axis=0)
    seglen = np.linalg.norm(seg, axis=1)
    cum = np.concatenate([[0.0], np.cumsum(seglen)])
    if cum[-1] == 0:
        return np.repeat(points[:1], n, axis=0)
    targets = np.linspace(0.0, cum[-1], n)
    k = np.clip(np.searchsorted(cum, targets, side="right") - 1, 0, len(seg) - 1)
    frac = (targets - cum[k]) / np.where(seglen[k] == 0, 1.0, seglen[k])
    return points[k] + frac[:, None] * seg[k]


def _presence(rng, n: int, duration: float) -> np.ndarray:
    length = rng.uniform(0.0, 0.4 * duration, n)
    start = rng.uniform(0.0, 1.0, n) * (duration - length)
    return np.stack([start, start + length], axis=1).astype(np.float32)


def generate_aerial_scene(seed, n_points, grid=(4, 4), n_views=16, altitude=50.0, image_size=(256, 256),
                          fov=None, duration=None) -> SceneDataset:
    """Downward cameras on a serpentine path over a noisy ground slab."""
    rows, cols = grid
    if n_points < 1 or n_views < 1 or altitude <= 0 or rows < 1 or cols < 1:
        raise ParameterError("n_points, n_views, altitude and grid must be positive")
    rng = _stream(seed, 0)
    fov = 2.0 * math.atan(0.6) if fov is None else float(fov)
    cell = float(altitude)
    density = rng.uniform(0.5, 1.5, size=rows * cols)
    per_cell = rng.multinomial(n_points, density / density.sum())
    xs, ys = [], []
    for k in range(rows * cols):
        r, c = divmod(k, cols)
        xs.append(rng.uniform(c * cell, (c + 1) * cell, per_cell[k]))
        ys.append(rng.uniform(r * cell, (r + 1) * cell, per_cell[k]))
    z = rng.uniform(0.0, 0.02 * altitude, n_points)
    positions = np.stack([np.concatenate(xs), np.concatenate(ys), z], axis=1).astype(np.float32)
    timestamps, profile = None, PROFILE_3DGS
    if duration is not None:
        if duration <= 0:
            raise ParameterError("duration must be > 0")
        timestamps, profile = _presence(rng, n_points, float(duration)), PROFILE_4DGS
    centres = []
    for r in range(rows):
        order = range(cols) if r % 2 == 0 else range(cols - 1, -1, -1)
        centres.extend([(c + 0.5) * cell, (r + 0.5) * cell] for c in order)
    path = _arclength_resample(np.array(centres), n_views)
    down = np.array([[1.0, 0.0, 0.0], [0.0, -1.0, 0.0], [0.0, 0.0, -1.0]])
    times = np.linspace(0.0, float(duration), n_views) if duration is not None else None
    width, height = image_size
    views = [CameraView(i, np.array([path[i, 0], path[i, 1], altitude]), down, fov, fov, 0.05 * altitude,
                        4.0 * altitude, width, height, None if times is None else float(times[i]))
             for i in range(n_views)]
    return SceneDataset(PointCloud(positions, timestamps), views, profile)


def _heading(direction) -> np.ndarray:
    fwd = np.asarray(direction, dtype=np.float64)
    n = np.linalg.norm(fwd)
    if n == 0:
        raise ParameterError("camera heading must be non-zero")
    fwd = fwd / n
    right = np.cross(fwd, np.array([0.0, 0.0, 1.0]))
    rn = np.linalg.norm(right)
    right = np.array([1.0, 0.0, 0.0]) if rn < 1e-12 else right / rn
    r = np.stack([right, np.cross(fwd, right), fwd], axis=1)
    u, _, vt = np.linalg.svd(r)
    return u @ vt


def generate_street_scene(seed, n_points, trajectory_waypoints, n_views, corridor_radius=8.0,
                          background_fraction=0.05, image_size=(256, 256), far_scale=0.12,
                          duration=None) -> SceneDataset:
    """Corridor of points along a polyline plus a distant background shell."""
    wps = np.asarray([p.as_array() if isinstance(p, Point3) else np.asarray(p, dtype=np.float64)
                      for p in trajectory_waypoints])
    if wps.ndim != 2 or wps.shape[1] != 3 or len(wps) < 2:
        raise ParameterError("need at least 2 waypoints of shape (3,)")
    if n_points < 1 or n_views < 1 or not (0.0 <= background_fraction < 1.0):
        raise ParameterError("bad street-scene size arguments")
    rng = _stream(seed, 0)
    seg = np.diff(wps, axis=0)
    seglen = np.linalg.norm(seg, axis=1)
    total = seglen.sum()
    if total == 0:
        raise ParameterError("trajectory has zero length")
    n_bg = int(round(background_fraction * n_points))
    n_corr = n_points - n_bg
    sidx = rng.choice(len(seg), size=n_corr, p=seglen / total)
    t = rng.uniform(0.0, 1.0, n_corr)
    up = np.array([0.0, 0.0, 1.0])
    dirs = seg[sidx] / seglen[sidx][:, None]
    side = np.cross(dirs, up)
    sn = np.linalg.norm(side, axis=1, keepdims=True)
    side = side / np.where(sn < 1e-12, 1.0, sn)
    side[sn[:, 0] < 1e-12] = [1.0, 0.0, 0.0]
    lat = rng.normal(0.0, corridor_radius / 2.5, n_corr)
    vert = np.abs(rng.normal(0.0, corridor_radius / 5.0, n_corr))
    corridor = (wps[sidx] + t[:, None] * seg[sidx]) + lat[:, None] * side + vert[:, None] * up
    centre = wps.mean(axis=0)
    theta = rng.uniform(0.0, 2.0 * math.pi, n_bg)
    rad = 0.15 * total + rng.uniform(10.0, 30.0, n_bg) * corridor_radius
    bz = rng.uniform(0.0, 10.0 * corridor_radius, n_bg)
    shell = np.stack([centre[0] + rad * np.cos(theta), centre[1] + rad * np.sin(theta), bz], axis=1)
    positions = np.concatenate([corridor, shell]).astype(np.float32)
    timestamps, profile = None, PROFILE_3DGS
    if duration is not None:
        if duration <= 0:
            raise ParameterError("duration must be > 0")
        timestamps, profile = _presence(rng, n_points, float(duration)), PROFILE_4DGS
    cam = _arclength_resample(wps, n_views)
    far = far_scale * total + 30.0 * corridor_radius
    times = np.linspace(0.0, float(duration), n_views) if duration is not None else None
    width, height = image_size
    views = []
    for i in range(n_views):
        j = min(i + 1, n_views - 1)
        h = cam[j] - cam[i] if j != i else cam[i] - cam[i - 1]
        if np.linalg.norm(h) < 1e-12:
            h = seg[0]
        views.append(CameraView(i, cam[i], _heading(h), 1.2, 1.2, 0.5, far, width, height,
                                None if times is None else float(times[i])))
    return SceneDataset(PointCloud(positions, timestamps), views, profile)


# ---------------------------------------------------------------------------
# trainable Gaussian state


SH_COEFFS = 16
# per-attribute Adam learning rates (standard 3DGS defaults; means scaled by
# the scene extent as in the 3DGS reference trainer)
DEFAULT_LR = {"means": 1.6e-4, "scales": 5e-3, "quats": 1e-3, "opacities": 5e-2, "sh0": 2.5e-3,
              "shN": 2.5e-3 / 20.0}


def lr_table(scene_extent: float = 1.0, lr: dict | None = None) -> np.ndarray:
    """Per-(plane, lane) learning rates of the 60-float parameter row."""
    lr = dict(DEFAULT_LR, **(lr or {}))
    t = np.zeros(60, dtype=np.float32)
    t[0:3] = lr["means"] * scene_extent
    t[3] = lr["opacities"]
    t[4:7] = lr["scales"]
    t[8:12] = lr["quats"]
    t[12:15] = lr["sh0"]
    t[15:60] = lr["shN"]
    return t


def init_gaussians(cloud: PointCloud, seed: int, spacing: float) -> np.ndarray:
    """Plane-major float4 parameters [15, S, 4] for the points of `cloud`.

    Attribute draws (stream SeedSequence([seed, 4]), in this order):
    scale factors U(0.5, 1.5) (S, 3); quaternions N(0, 1) (S, 4) normalised;
    opacity U(0.1, 0.9) -> logit; sh0 N(0, 0.3) (S, 3); shN N(0, 0.03) (S, 45).
    log_scale = log(spacing * f) on x, y and log(0.3 * spacing * f) on z.
    """
    return init_gaussians_rows(cloud, seed, spacing, None)


def init_gaussians_rows(cloud: PointCloud, seed: int, spacing: float, rows: np.ndarray | None) -> np.ndarray:
    """init_gaussians restricted to the points `rows` (ascending indices into
    `cloud`; None = all): [15, len(rows), 4].  Every draw of the stream is
    made in row blocks (a block draw continues the stream exactly like one
    (S, k) draw), and only the selected rows are kept, so a rank of a
    50M-200M point scene materialises its own shard and no float64 [S, k]
    array (bench.py, one process per GPU)."""
    S = len(cloud)
    rng = _stream(seed, 4)
    sel = np.arange(S, dtype=np.int64) if rows is None else np.asarray(rows, dtype=np.int64)
    if len(sel) and (np.any(np.diff(sel) <= 0) or sel[0] < 0 or sel[-1] >= S):
        raise ParameterError("rows must be ascending unique point indices")
    n = len(sel)
    out = np.zeros((15, n, 4), dtype=np.float32)
    step = 1 << 22
    blocks = [(r0, min(S, r0 + step)) for r0 in range(0, S, step)]
    # output slice of every block: sel[lo:hi] lies in [r0, r1)
    cuts = np.searchsorted(sel, [b[0] for b in blocks] + [S])

    def each_block(draw):
        for k, (r0, r1) in enumerate(blocks):
            vals = draw(r1 - r0)
            lo, hi = cuts[k], cuts[k + 1]
            yield lo, hi, (vals if rows is None else vals[sel[lo:hi] - r0])

    out[0, :, :3] = np.asarray(cloud.positions) if rows is None else np.asarray(cloud.positions)[sel]
    for lo, hi, f in each_block(lambda m: rng.uniform(0.5, 1.5, size=(m, 3))):
        ls = np.log(spacing * f)
        ls[:, 2] = np.log(0.3 * spacing * f[:, 2])
        out[1, lo:hi, :3] = ls
    for lo, hi, quat in each_block(lambda m: rng.normal(0.0, 1.0, size=(m, 4))):
        out[2, lo:hi] = quat / np.linalg.norm(quat, axis=1, keepdims=True)
    for lo, hi, op in each_block(lambda m: rng.uniform(0.1, 0.9, size=m)):
        out[0, lo:hi, 3] = np.log(op / (1.0 - op))
    sh0 = np.zeros((n, 3), dtype=np.float64)
    for lo, hi, v in each_block(lambda m: rng.normal(0.0, 0.3, size=(m, 3))):
        sh0[lo:hi] = v
    for lo, hi, shn in each_block(lambda m: rng.normal(0.0, 0.03, size=(m, 45))):
        sh = np.concatenate([sh0[lo:hi], shn], axis=1).astype(np.float32)  # f = 3k + channel
        out[3:15, lo:hi] = sh.reshape(hi - lo, 12, 4).transpose(1, 0, 2)
    return out


def synthetic_gt(seed: int, n_views: int, width: int, height: int) -> np.ndarray:
    """Ground-truth images u8 [n_views, H, W, 3] from SeedSequence([seed, 5])."""
    rng = _stream(seed, 5)
    return rng.integers(0, 256, size=(n_views, height, width, 3), dtype=np.uint8)


def synthetic_gt_views(seed: int, view_ids, width: int, height: int) -> np.ndarray:
    """Ground truth of selected views only, u8 [len(view_ids), H, W, 3]; view v
    from SeedSequence([seed, 5, v]) (large configurations, where materialising
    every view is wasteful)."""
    out = np.empty((len(view_ids), height, width, 3), dtype=np.uint8)
    for k, v in enumerate(view_ids):
        rng = np.random.default_rng(np.random.SeedSequence([int(seed), 5, int(v)]))
        out[k] = rng.integers(0, 256, size=(height, width, 3), dtype=np.uint8)
    return out


def mean_spacing(altitude: float, grid, n_points: int) -> float:
    rows, cols = grid
    return float(altitude) * math.sqrt(rows * cols / float(n_points))
