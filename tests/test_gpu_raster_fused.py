"""K3 + L + K4 fused (bs_raster_fwd_bwd, csrc/raster.cu raster_fused_kernel)
against the two-kernel path (bs_raster_fwd + bs_raster_bwd): identical image,
transmittance, contributor counts and losses; G_SP within atomic-order
tolerance -- at C1 (both backgrounds, and with the kept list forced to wrap
for every warp) and on a full C2 batch."""

import numpy as np
import pytest
import torch

from paper_2512_20017_b200 import scenes
from paper_2512_20017_b200.culling import zorder_group
from paper_2512_20017_b200.trainer import SplatTrainer

from _scene import c1_setup

pytestmark = pytest.mark.gpu

REL = 1e-5


def _run(make, batch, fused):
    tr = make()
    tr.raster_fused = fused
    tr.keep_raster_aux = True  # T and n_contrib compared below
    losses = tr.step(batch).cpu().numpy()
    n = tr.last["n_rows"]
    npx = len(batch) * tr.H * tr.W
    gf = tr.gsp_floats
    return (losses, tr.last["image"][: npx * 3].cpu().numpy(), tr.last["final_T"][:npx].cpu().numpy(),
            tr.last["n_contrib"][:npx].cpu().numpy(), tr.last["gsp"][: n * gf].cpu().numpy().reshape(-1, gf),
            tr.gsp_wire_floats)


def _compare(make, batch):
    a = _run(make, batch, True)
    b = _run(make, batch, False)
    for x, y in zip(a[:4], b[:4]):
        assert np.array_equal(x, y)
    wire = a[5]
    assert not a[4][:, wire:].any()
    scale = np.abs(b[4][:, :wire]).max(axis=0) + 1e-30
    err = (np.abs(a[4][:, :wire] - b[4][:, :wire]) / scale).max(axis=0)
    assert (err <= REL).all(), err
    return err


@pytest.mark.parametrize("model", ["3dgs", "2dgs"])
@pytest.mark.parametrize("bg", [(0.0, 0.0, 0.0), (0.2, 0.5, 0.9)])
def test_fused_matches_two_kernels_c1(cuda, bg, model):
    ds, params, gb, aabb, gt = c1_setup()
    _compare(lambda: SplatTrainer(params, gb, aabb, ds.views, gt=gt, sh_degree=3, bg=bg, model=model), [0, 2, 5, 7])


@pytest.mark.parametrize("model", ["3dgs", "2dgs"])
def test_fused_wrapped_lists_fall_back(cuda, model):
    """Large splats: every warp keeps far more splats than its shared-memory
    list holds, so the fused kernel's backward takes the chunked global walk."""
    ds, params, gb, aabb, gt = c1_setup()
    params = params.copy()
    params[1, :, :3] += np.float32(1.5)
    _compare(lambda: SplatTrainer(params, gb, aabb, ds.views, gt=gt, sh_degree=3, model=model), [1, 6])


def test_fused_matches_two_kernels_c2(cuda):
    ds = scenes.generate_aerial_scene(1, 1_000_000, (1, 1), 8, 50.0, (1920, 1080))
    g = zorder_group(ds.cloud, G=2048)
    params = scenes.init_gaussians(g.sorted_cloud, 1, scenes.mean_spacing(50.0, (1, 1), 1_000_000))
    gt = scenes.synthetic_gt(1, 8, 1920, 1080)
    err = _compare(lambda: SplatTrainer(params, g.group_begin(), g.aabbs.reshape(-1, 6), ds.views, gt=gt),
                   [0, 3, 4, 7])
    print("C2 G_SP max rel diff per component", err)


def test_fused_matches_two_kernels_c3(cuda):
    ds = scenes.generate_aerial_scene(2, 2_000_000, (1, 1), 8, 50.0, (1920, 1080))
    g = zorder_group(ds.cloud, G=2048)
    params = scenes.init_gaussians(g.sorted_cloud, 2, scenes.mean_spacing(50.0, (1, 1), 2_000_000))
    gt = scenes.synthetic_gt(2, 8, 1920, 1080)
    err = _compare(lambda: SplatTrainer(params, g.group_begin(), g.aabbs.reshape(-1, 6), ds.views, gt=gt,
                                        model="2dgs"), [1, 2, 5, 6])
    print("C3 G_SP max rel diff per component", err.max())


def test_fused_without_aux_outputs_c1(cuda):
    """The training step's default skips the fused kernel's T / n_contrib
    stores (8 B per pixel); image, losses and G_SP are unaffected."""
    ds, params, gb, aabb, gt = c1_setup()
    outs = []
    for aux in (True, False):
        tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, sh_degree=3)
        tr.keep_raster_aux = aux
        losses = tr.step([0, 2, 5, 7]).cpu().numpy()
        n, npx = tr.last["n_rows"], 4 * tr.H * tr.W
        outs.append((losses, tr.last["image"][: npx * 3].cpu().numpy(),
                     tr.last["gsp"][: n * tr.gsp_floats].cpu().numpy().reshape(n, -1)))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    scale = np.abs(outs[0][2]).max(axis=0) + 1e-30
    assert ((np.abs(outs[0][2] - outs[1][2]) / scale).max() <= REL)
