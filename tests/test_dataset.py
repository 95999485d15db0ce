"""splatsched-v1 dataset files (dataset.py) against files written by the
unmodified reference (tests/golden/dataset_v1, make_dataset_golden.py), the
gaussians/images extensions, and the sharded ground-truth store."""

import filecmp
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_20017_b200 import dataset as dsio
from paper_2512_20017_b200 import scenes
from paper_2512_20017_b200.status import DatasetFormatError, DatasetVersionError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "dataset_v1")


def _cases():
    return {
        "aerial": scenes.generate_aerial_scene(3, 60, (2, 2), 3, 25),
        "temporal": scenes.generate_aerial_scene(4, 40, (1, 2), 4, 20, duration=5.0),
        "street": scenes.generate_street_scene(11, 50, [(0, 0, 2), (40, 0, 2), (40, 30, 2)], 4),
    }


@pytest.mark.parametrize("name", ["aerial", "temporal", "street"])
def test_reference_files_roundtrip_byte_identical(tmp_path, name):
    ds = _cases()[name]
    assert dsio.load_dataset(os.path.join(GOLD, name)) == ds
    dsio.save_dataset(ds, str(tmp_path))
    for fn in ("dataset.json", "points.bin"):
        assert filecmp.cmp(tmp_path / fn, os.path.join(GOLD, name, fn), shallow=False), fn


def test_format_errors(tmp_path):
    ds = _cases()["aerial"]
    dsio.save_dataset(ds, str(tmp_path))
    blob = (tmp_path / "points.bin").read_bytes()
    (tmp_path / "points.bin").write_bytes(blob[: len(blob) // 2])
    with pytest.raises(DatasetFormatError) as e:
        dsio.load_dataset(str(tmp_path))
    assert e.value.byte_offset is not None
    (tmp_path / "points.bin").write_bytes(b"XXXX" + blob[4:])
    with pytest.raises(DatasetFormatError):
        dsio.load_dataset(str(tmp_path))
    (tmp_path / "points.bin").write_bytes(blob)
    h = tmp_path / "dataset.json"
    h.write_text(h.read_text().replace("splatsched-v1", "v999"))
    with pytest.raises(DatasetVersionError):
        dsio.load_dataset(str(tmp_path))


def test_gaussian_and_image_extensions(tmp_path):
    ds = _cases()["aerial"]
    dsio.save_dataset(ds, str(tmp_path))
    rng = np.random.default_rng(0)
    p = rng.normal(size=(15, 60, 4)).astype(np.float32)
    m, v = rng.normal(size=p.shape).astype(np.float32), rng.uniform(size=p.shape).astype(np.float32)
    dsio.save_gaussians(str(tmp_path), p, m, v, sh_degree=3, step=7)
    imgs = rng.integers(0, 256, (3, 20, 30, 3), dtype=np.uint8)
    dsio.save_images(str(tmp_path), imgs)
    assert dsio.load_dataset(str(tmp_path)) == ds  # extensions leave the v1 content intact
    p2, m2, v2, meta = dsio.load_gaussians(str(tmp_path))
    assert np.array_equal(p2, p) and np.array_equal(m2, m) and np.array_equal(v2, v)
    assert meta["step"] == 7 and meta["sh_degree"] == 3
    assert np.array_equal(dsio.open_images(str(tmp_path)), imgs)
    blob = (tmp_path / "images.bin").read_bytes()
    (tmp_path / "images.bin").write_bytes(blob[:-5])
    with pytest.raises(DatasetFormatError):
        dsio.open_images(str(tmp_path))


def test_gt_store_single_rank():
    imgs = np.arange(4 * 5 * 6 * 3, dtype=np.uint8).reshape(4, 5, 6, 3)
    store = dsio.GTStore(imgs, [0, 1, 2, 3], np.zeros(4, dtype=np.int64), 0, pin=False)
    out = torch.empty((2, 5, 6, 3), dtype=torch.uint8)
    store.fetch(np.array([0, 0]), [3, 1], out)
    assert np.array_equal(out.numpy(), imgs[[3, 1]])
    with pytest.raises(Exception):
        dsio.GTStore(imgs, [0], np.ones(4, dtype=np.int64), 0, pin=False)


def _gt_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_20017_b200.exchange import SplatExchange

        rng = np.random.default_rng(5)
        imgs = rng.integers(0, 256, (8, 7, 9, 3), dtype=np.uint8)
        owner = np.array([0, 1, 0, 1, 1, 0, 0, 1])
        store = dsio.GTStore(imgs, np.flatnonzero(owner == rank), owner, rank, pin=False)
        batch = [5, 2, 7, 4]
        W = np.array([1, 0, 0, 1])  # views 5 (owner 0) -> rank 1, 7 (owner 1) -> rank 0
        out = torch.zeros((2, 7, 9, 3), dtype=torch.uint8)
        store.fetch(W, batch, out, comm=SplatExchange())
        mine = [batch[j] for j in range(4) if W[j] == rank]
        q.put((rank, np.array_equal(out.numpy(), imgs[mine]), store.remote_bytes))
    finally:
        dist.destroy_process_group()


def test_gt_store_two_ranks_fetch_remote():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gt_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((item[0], item) for item in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] and res[1][1]
    assert res[0][2] == res[1][2] == 7 * 9 * 3  # one image arrives at each rank
