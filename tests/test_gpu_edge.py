"""Edge cases of the GPU training step: views that see no point (empty splat
sets, alone and inside a batch), the largest batch (32 views, one u32
visibility mask), image sizes that are not a multiple of the 16-pixel tile
(and smaller than one tile), ragged point groups, and both splat models --
each against the CPU oracle (bit-exact splat rows and tile lists, images and
gradients to the fp32 tolerance)."""

import numpy as np
import pytest
import torch

from _scene import c1_setup, oracle_view_pipeline
from paper_2512_20017_b200 import scenes
from paper_2512_20017_b200.scenes import CameraView
from paper_2512_20017_b200.trainer import AdamConfig, SplatTrainer, camera_bytes

pytestmark = pytest.mark.gpu
IMG_TOL = 1e-4
GRAD_REL = 1e-4


def _away(view, k):
    """The same camera moved far outside the scene: sees nothing."""
    return CameraView(k, view.position + np.array([1e5, 1e5, 0.0]), view.rotation, view.fov_x, view.fov_y,
                      view.near, view.far, view.width, view.height, view.time)


def _check_views(tr, ds, params, gb, aabb, gt, batch, model="3dgs"):
    H, W = tr.H, tr.W
    spf, gpf = (24, 16) if model == "2dgs" else (12, 12)
    n = tr.last["n_rows"]
    sp = tr.last["sp"][: n * spf].cpu().numpy().reshape(-1, spf)
    img = tr.last["image"][: len(batch) * H * W * 3].cpu().numpy().reshape(len(batch), H, W, 3)
    gsp = tr.last["gsp"][: n * gpf].cpu().numpy().reshape(-1, gpf)[:, : (15 if model == "2dgs" else 9)]
    rows = tr.last["rows_per_view"]
    row0 = np.concatenate([[0], np.cumsum(rows)])
    for s, v in enumerate(batch):
        ref = oracle_view_pipeline(params, gb, aabb, ds.views[v], camera_bytes([ds.views[v]]), gt[v], model=model)
        assert rows[s] == len(ref["idx"])
        assert np.array_equal(sp[row0[s]:row0[s + 1]].view(np.uint32), ref["sp"].view(np.uint32))
        assert np.abs(img[s] - ref["img"]).max() <= IMG_TOL
        if len(ref["idx"]):
            g = gsp[row0[s]:row0[s + 1]]
            scale = np.abs(ref["gsp"]).max(axis=0) + 1e-30
            assert ((np.abs(g - ref["gsp"]) / scale).max(axis=0) <= GRAD_REL).all()


@pytest.mark.parametrize("model", ["3dgs", "2dgs"])
def test_empty_view_alone_and_in_batch(cuda, model):
    ds, params, gb, aabb, gt = c1_setup()
    ds.views.append(_away(ds.views[0], len(ds.views)))
    gt = np.concatenate([gt, gt[:1]])
    tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, adam=AdamConfig(scenes.lr_table(50.0)), model=model)
    empty = len(ds.views) - 1
    losses = tr.step([empty]).cpu().numpy()  # nothing visible anywhere
    assert tr.last["n_rows"] == 0 and tr.last["n_inst"] == 0
    np.testing.assert_allclose(losses[0], np.abs(gt[empty].astype(np.float64) / 255.0).mean(), atol=1e-6)
    np.testing.assert_array_equal(tr.params.cpu().numpy(), params)  # zero gradient: Adam leaves params unchanged
    tr2 = SplatTrainer(params, gb, aabb, ds.views, gt=gt, adam=AdamConfig(scenes.lr_table(50.0)), model=model)
    batch = [1, empty, 4]
    tr2.step(batch)
    torch.cuda.synchronize()
    _check_views(tr2, ds, params, gb, aabb, gt, batch, model)


def test_max_batch_32_views(cuda):
    ds, params, gb, aabb, gt = c1_setup(n_views=32, image_size=(64, 48))
    tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, adam=AdamConfig(scenes.lr_table(50.0)))
    batch = list(range(32))[::-1]
    tr.step(batch)
    torch.cuda.synchronize()
    _check_views(tr, ds, params, gb, aabb, gt, batch)
    with pytest.raises(ValueError):
        tr.step(list(range(32)) + [0])


@pytest.mark.parametrize("size", [(37, 21), (9, 7), (16, 16), (300, 17)])
def test_image_sizes_off_the_tile_grid(cuda, size):
    ds, params, gb, aabb, gt = c1_setup(image_size=size, n_points=3001)  # ragged last group (3001 % 256)
    tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, adam=AdamConfig(scenes.lr_table(50.0)))
    batch = [0, 5]
    tr.step(batch)
    torch.cuda.synchronize()
    _check_views(tr, ds, params, gb, aabb, gt, batch)
