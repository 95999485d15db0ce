"""Dataset storage and ground-truth loading of the training path.

File format: the reference's ``splatsched-v1`` directory
(/root/reference/pkg/src/splatsched/scene.py:468-578) --
``dataset.json`` (version, profile, n_points, temporal, views) and
``points.bin`` (magic ``SSPC``, u32 count, f32 positions [, f32 presence]).
``save_dataset`` writes it byte for byte as the reference does and
``load_dataset`` reads the reference's files (same errors: DatasetFormatError
with the byte offset, DatasetVersionError).  Two optional files extend it for
training, declared under ``"extensions"`` in the header (a key the reference
loader ignores):

  gaussians.bin  magic ``SSGS``, u32 n_points, u32 planes (15), then the
                 plane-major float32 parameters [15][n][4]
                 (include/splat_b200.h parameter layout, Z-order sorted)
                 and optionally the two Adam moments in the same layout
  images.bin     magic ``SSIM``, u32 n_views, u32 height, u32 width, then
                 u8 RGB [n_views][H][W][3] in view-id order (pre-decoded
                 ground truth)

Ground truth at train time: ``GTStore`` keeps the images
of the views this rank owns (image_ownership of the offline partition,
partition.py:537-541) pre-decoded in pinned host memory -- the dataset is
spread over the ranks' host memory instead of replicated.  Per step each
rank needs the views the online placement W assigns to it: owned ones are
copied host->device directly; the rest are sent device-to-device by their
owners in one all_to_all (sizes follow from W and the ownership map, which
every rank holds, so no size exchange).
"""

from __future__ import annotations

import json
import os
import struct

import numpy as np

from .scenes import CameraView, PointCloud, SceneDataset, WorkloadProfile
from .status import DatasetFormatError, DatasetVersionError, ParameterError

FORMAT_VERSION = "splatsched-v1"
HEADER_NAME = "dataset.json"
POINTS_NAME = "points.bin"
POINTS_MAGIC = b"SSPC"
GAUSSIANS_NAME = "gaussians.bin"
GAUSSIANS_MAGIC = b"SSGS"
IMAGES_NAME = "images.bin"
IMAGES_MAGIC = b"SSIM"
PARAM_PLANES = 15


def _view_to_json(v: CameraView) -> dict:
    return {"id": v.id, "position": [float(c) for c in v.position], "rotation": [float(c) for c in v.rotation.reshape(-1)],
            "fov_x": v.fov_x, "fov_y": v.fov_y, "near": v.near, "far": v.far, "width": v.width,
            "height": v.height, "time": v.time}


def _view_from_json(d: dict) -> CameraView:
    return CameraView(int(d["id"]), np.array(d["position"], dtype=np.float64),
                      np.array(d["rotation"], dtype=np.float64).reshape(3, 3), float(d["fov_x"]), float(d["fov_y"]),
                      float(d["near"]), float(d["far"]), int(d["width"]), int(d["height"]),
                      None if d.get("time") is None else float(d["time"]))


def _header(dataset: SceneDataset, extensions: dict | None) -> dict:
    h = {
        "version": FORMAT_VERSION,
        "profile": {"name": dataset.profile.name, "splat_state_elements": dataset.profile.splat_state_elements,
                    "bytes_per_element": dataset.profile.bytes_per_element,
                    "culling_mode": dataset.profile.culling_mode},
        "n_points": len(dataset.cloud),
        "temporal": dataset.cloud.timestamps is not None,
        "points_file": POINTS_NAME,
        "views": [_view_to_json(v) for v in dataset.views],
    }
    if extensions:
        h["extensions"] = extensions
    return h


def _read_header(path: str) -> dict:
    try:
        with open(os.path.join(path, HEADER_NAME)) as f:
            header = json.load(f)
    except json.JSONDecodeError as e:
        raise DatasetFormatError(f"invalid JSON header: {e.msg}", e.pos) from e
    if header.get("version") != FORMAT_VERSION:
        raise DatasetVersionError(f"unsupported dataset version {header.get('version')!r}, "
                                  f"expected {FORMAT_VERSION!r}")
    return header


def _write_header(path: str, header: dict) -> None:
    with open(os.path.join(path, HEADER_NAME), "w") as f:
        json.dump(header, f, indent=1, sort_keys=True)


def save_dataset(dataset: SceneDataset, path: str) -> None:
    """dataset.json + points.bin in directory `path` (scene.py:503-528)."""
    os.makedirs(path, exist_ok=True)
    _write_header(path, _header(dataset, None))
    with open(os.path.join(path, POINTS_NAME), "wb") as f:
        f.write(POINTS_MAGIC)
        f.write(struct.pack("<I", len(dataset.cloud)))
        f.write(dataset.cloud.positions.astype("<f4").tobytes())
        if dataset.cloud.timestamps is not None:
            f.write(dataset.cloud.timestamps.astype("<f4").tobytes())


def load_dataset(path: str) -> SceneDataset:
    """Read a splatsched-v1 directory (scene.py:531-578)."""
    header = _read_header(path)
    prof = header["profile"]
    profile = WorkloadProfile(prof["name"], int(prof["splat_state_elements"]), int(prof["bytes_per_element"]),
                              prof["culling_mode"])
    n, temporal = int(header["n_points"]), bool(header["temporal"])
    with open(os.path.join(path, header.get("points_file", POINTS_NAME)), "rb") as f:
        blob = f.read()
    if blob[:4] != POINTS_MAGIC:
        raise DatasetFormatError("bad magic bytes in points file", 0)
    if len(blob) < 8:
        raise DatasetFormatError("points file truncated in header", len(blob))
    (count,) = struct.unpack_from("<I", blob, 4)
    if count != n:
        raise DatasetFormatError(f"point count {count} disagrees with header ({n})", 4)
    expected = 8 + count * 12 + (count * 8 if temporal else 0)
    if len(blob) != expected:
        raise DatasetFormatError(f"points file has {len(blob)} bytes, expected {expected}", min(len(blob), expected))
    positions = np.frombuffer(blob, dtype="<f4", count=count * 3, offset=8).reshape(count, 3).copy()
    timestamps = None
    if temporal:
        timestamps = np.frombuffer(blob, dtype="<f4", count=count * 2, offset=8 + count * 12).reshape(count, 2).copy()
    views = [_view_from_json(d) for d in header["views"]]
    return SceneDataset(PointCloud(positions, timestamps), views, profile)


def _add_extension(path: str, name: str, entry: dict) -> None:
    header = _read_header(path)
    ext = dict(header.get("extensions", {}))
    ext[name] = entry
    header["extensions"] = ext
    _write_header(path, header)


# ---------------------------------------------------------------- Gaussians


def save_gaussians(path: str, params: np.ndarray, exp_avg: np.ndarray | None = None,
                   exp_avg_sq: np.ndarray | None = None, sh_degree: int = 3, step: int = 0) -> None:
    """Plane-major parameters [15, n, 4] (+ Adam moments) of the dataset's
    Z-ordered points -> gaussians.bin, declared in dataset.json."""
    p = np.ascontiguousarray(params, dtype="<f4")
    if p.ndim != 3 or p.shape[0] != PARAM_PLANES or p.shape[2] != 4:
        raise ParameterError("params must be float32 [15, n, 4]")
    moments = exp_avg is not None and exp_avg_sq is not None
    with open(os.path.join(path, GAUSSIANS_NAME), "wb") as f:
        f.write(GAUSSIANS_MAGIC)
        f.write(struct.pack("<II", p.shape[1], PARAM_PLANES))
        f.write(p.tobytes())
        if moments:
            for m in (exp_avg, exp_avg_sq):
                f.write(np.ascontiguousarray(m, dtype="<f4").reshape(p.shape).tobytes())
    _add_extension(path, "gaussians", {"file": GAUSSIANS_NAME, "layout": "planes-15x4-f32", "n_points": int(p.shape[1]),
                                       "sh_degree": int(sh_degree), "adam_moments": bool(moments), "step": int(step)})


def load_gaussians(path: str):
    """(params, exp_avg | None, exp_avg_sq | None, meta) from gaussians.bin
    (memory-mapped; copy what you keep)."""
    header = _read_header(path)
    meta = header.get("extensions", {}).get("gaussians")
    if meta is None:
        raise DatasetFormatError("dataset has no gaussians extension", None)
    fn = os.path.join(path, meta["file"])
    size = os.path.getsize(fn)
    with open(fn, "rb") as f:
        head = f.read(12)
    if head[:4] != GAUSSIANS_MAGIC:
        raise DatasetFormatError("bad magic bytes in gaussians file", 0)
    if len(head) < 12:
        raise DatasetFormatError("gaussians file truncated in header", len(head))
    n, planes = struct.unpack_from("<II", head, 4)
    if planes != PARAM_PLANES or n != int(meta["n_points"]):
        raise DatasetFormatError(f"gaussians file declares {n} points x {planes} planes", 4)
    one = PARAM_PLANES * n * 4 * 4
    copies = 3 if meta.get("adam_moments") else 1
    if size != 12 + copies * one:
        raise DatasetFormatError(f"gaussians file has {size} bytes, expected {12 + copies * one}",
                                 min(size, 12 + copies * one))
    mm = np.memmap(fn, dtype="<f4", mode="r", offset=12, shape=(copies, PARAM_PLANES, n, 4))
    return mm[0], (mm[1] if copies == 3 else None), (mm[2] if copies == 3 else None), meta


# ---------------------------------------------------------------- images


def save_images(path: str, images: np.ndarray) -> None:
    """Pre-decoded ground truth u8 [n_views, H, W, 3] (view-id order)."""
    im = np.ascontiguousarray(images, dtype=np.uint8)
    if im.ndim != 4 or im.shape[3] != 3:
        raise ParameterError("images must be uint8 [n_views, H, W, 3]")
    with open(os.path.join(path, IMAGES_NAME), "wb") as f:
        f.write(IMAGES_MAGIC)
        f.write(struct.pack("<III", *im.shape[:3]))
        f.write(im.tobytes())
    _add_extension(path, "images", {"file": IMAGES_NAME, "shape": [int(x) for x in im.shape], "dtype": "u8"})


def open_images(path: str) -> np.ndarray:
    """Memory-mapped u8 [n_views, H, W, 3] ground truth of a dataset."""
    header = _read_header(path)
    meta = header.get("extensions", {}).get("images")
    if meta is None:
        raise DatasetFormatError("dataset has no images extension", None)
    fn = os.path.join(path, meta["file"])
    with open(fn, "rb") as f:
        head = f.read(16)
    if head[:4] != IMAGES_MAGIC:
        raise DatasetFormatError("bad magic bytes in images file", 0)
    if len(head) < 16:
        raise DatasetFormatError("images file truncated in header", len(head))
    n, h, w = struct.unpack_from("<III", head, 4)
    if [n, h, w, 3] != list(meta["shape"]):
        raise DatasetFormatError(f"images file declares {n}x{h}x{w}", 4)
    size, want = os.path.getsize(fn), 16 + n * h * w * 3
    if size != want:
        raise DatasetFormatError(f"images file has {size} bytes, expected {want}", min(size, want))
    return np.memmap(fn, dtype=np.uint8, mode="r", offset=16, shape=(n, h, w, 3))


# ---------------------------------------------------------------- GT store


class GTStore:
    """Ground truth of the views `owned` by this rank, pre-decoded in pinned
    host memory.  `fetch(W, batch, out)` fills `out`
    [slots, H, W, 3] (device) with the views W assigns to this rank, in the
    order of W's positions; owned views are copied host->device, the others
    arrive from their owners through one all_to_all (comm: SplatExchange or
    None for a single rank, which must own every view it renders)."""

    def __init__(self, images: np.ndarray, owned, owner_of: np.ndarray, rank: int = 0, pin: bool = True):
        import torch

        self.owner_of = np.asarray(owner_of, dtype=np.int64)
        self.rank = int(rank)
        self.owned = np.array(sorted(int(v) for v in owned), dtype=np.int64)
        if np.any(self.owner_of[self.owned] != self.rank):
            raise ParameterError("owned views disagree with the ownership map")
        self.shape = tuple(int(x) for x in images.shape[1:])
        self.slot_of = {int(v): k for k, v in enumerate(self.owned)}
        host = torch.from_numpy(np.ascontiguousarray(images[self.owned]))
        self.host = host.pin_memory() if pin and torch.cuda.is_available() else host
        self.h2d_bytes = 0
        self.remote_bytes = 0

    @classmethod
    def from_dataset(cls, path: str, owner_of, rank: int = 0, pin: bool = True):
        owner_of = np.asarray(owner_of, dtype=np.int64)
        return cls(open_images(path), np.flatnonzero(owner_of == rank), owner_of, rank, pin)

    def _local(self, v: int):
        return self.host[self.slot_of[int(v)]]

    def fetch(self, W: np.ndarray, batch, out, comm=None):
        import torch

        W = np.asarray(W, dtype=np.int64)
        batch = [int(v) for v in batch]
        mine = [j for j in range(len(batch)) if W[j] == self.rank]
        if out.shape[0] < len(mine):
            raise ParameterError("output holds fewer slots than the views placed on this rank")
        nb = int(np.prod(self.shape))
        remote = []
        for slot, j in enumerate(mine):
            v = batch[j]
            if self.owner_of[v] == self.rank:
                out[slot].copy_(self._local(v), non_blocking=True)
                self.h2d_bytes += nb
            else:
                remote.append((slot, v))
        if comm is None:
            if remote:
                raise ParameterError(f"views {[v for _, v in remote]} are not stored on this single rank")
            return out
        world = comm.world
        # every rank derives the same transfer list from (W, ownership)
        send = [[] for _ in range(world)]
        recv = [[] for _ in range(world)]
        for j, v in enumerate(batch):
            o, d = int(self.owner_of[v]), int(W[j])
            if o == d:
                continue
            if o == self.rank:
                send[d].append(v)
            if d == self.rank:
                recv[o].append(v)
        dev = out.device
        sbuf = torch.empty((sum(len(x) for x in send),) + self.shape, dtype=torch.uint8, device=dev)
        k = 0
        for d in range(world):
            for v in send[d]:
                sbuf[k].copy_(self._local(v), non_blocking=True)
                self.h2d_bytes += nb
                k += 1
        rows_s = [len(x) for x in send]
        rows_r = [len(x) for x in recv]
        rbuf = comm._a2a(sbuf.reshape(-1), rows_s, rows_r, nb)
        self.remote_bytes += rbuf.numel()
        at = {}
        k = 0
        for o in range(world):
            for v in recv[o]:
                at[v] = k
                k += 1
        for slot, v in remote:
            out[slot].copy_(rbuf[at[v]].view(self.shape))
        return out
