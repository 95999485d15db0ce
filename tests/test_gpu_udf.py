"""GPU parity of the UDF protocol:
pts_culling / pts_splatting / image_render as torch.autograd.Functions over
the C ABI, against the CPU oracle of the same view.

Tolerances as tests/test_gpu_parity.py: ids and splat rows bit-exact, image
max-abs <= 1e-4, parameter gradients <= 1e-4 x per-(plane, lane) max."""

import numpy as np
import pytest
import torch

from paper_2512_20017_b200 import image_render, pts_culling, pts_splatting
from paper_2512_20017_b200.trainer import camera_bytes

from _scene import c1_setup, oracle_view_pipeline

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
GRAD_REL = 1e-4
GRAD_REL_2DGS = 1e-4


@pytest.fixture(scope="module")
def c1(cuda):
    return c1_setup()


def _pc(params, dev):
    S = params.shape[1]
    P = torch.as_tensor(params, device=dev)
    return {
        "xyz": P[0, :, :3].clone().requires_grad_(True),
        "opacity": P[0, :, 3:4].clone().requires_grad_(True),
        "scaling": P[1, :, :3].clone().requires_grad_(True),
        "rotation": P[2].clone().requires_grad_(True),
        "sh": P[3:15].permute(1, 0, 2).reshape(S, 16, 3).clone().requires_grad_(True),
    }


def _grads_as_planes(PC, S):
    g = np.zeros((15, S, 4), dtype=np.float32)
    g[0, :, :3] = PC["xyz"].grad.cpu().numpy()
    g[0, :, 3] = PC["opacity"].grad.cpu().numpy()[:, 0]
    g[1, :, :3] = PC["scaling"].grad.cpu().numpy()
    g[2] = PC["rotation"].grad.cpu().numpy()
    g[3:15] = PC["sh"].grad.cpu().numpy().reshape(S, 12, 4).transpose(1, 0, 2)
    return g


@pytest.mark.parametrize("model", ["3dgs", "2dgs"])
def test_udf_pipeline_matches_oracle(c1, cuda, model):
    ds, params, gb, aabb, gt = c1
    S = params.shape[1]
    for v in (0, 5):
        view = ds.views[v]
        ref = oracle_view_pipeline(params, gb, aabb, view, camera_bytes([view]), gt[v], model=model)
        PC = _pc(params, cuda)
        ids = pts_culling(view, PC)
        assert np.array_equal(ids.cpu().numpy(), ref["idx"])
        SP = pts_splatting(view, PC, ids, sh_degree=3, model=model)
        width = 24 if model == "2dgs" else 12
        rows = torch.cat([SP["means2d"], SP["opacities"][:, None]], 1)
        assert rows.shape == (len(ref["idx"]), 3)
        from paper_2512_20017_b200.udf import pack_splats

        sp = pack_splats(SP).detach().cpu().numpy()
        assert sp.shape[1] == width
        ref_sp = ref["sp"].copy()
        if model == "2dgs":
            ref_sp[:, 21] = 0.0  # pad
        assert np.array_equal(sp.view(np.uint32), ref_sp.view(np.uint32)), "splat rows not bit-exact"
        img = image_render(view, SP)
        assert np.abs(img.detach().cpu().numpy() - ref["img"]).max() <= IMG_TOL
        loss = (img - torch.as_tensor(gt[v], device=cuda).float() / 255.0).abs().mean()
        assert abs(loss.item() - ref["loss"]) <= 1e-5
        loss.backward()
        g = _grads_as_planes(PC, S)
        g_ref = ref["gparams"]
        scale = np.abs(g_ref).reshape(15, -1, 4).max(axis=1) + 1e-30
        err = np.abs(g - g_ref).max(axis=1) / scale
        if model == "2dgs":
            err[1, 2:] = 0.0  # third scale / pad: unused by surfels (both zero)
        err[1, 3] = 0.0
        assert (err <= (GRAD_REL_2DGS if model == "2dgs" else GRAD_REL)).all(), err.max()


def test_udf_temporal_culling(c1, cuda):
    ds, params, gb, aabb, gt = c1
    S = params.shape[1]
    PC = _pc(params, cuda)
    rng = np.random.default_rng(4)
    t0 = rng.uniform(0, 1, S).astype(np.float32)
    pres = np.stack([t0, t0 + 0.3], 1).astype(np.float32)
    PC["presence"] = torch.as_tensor(pres, device=cuda)
    view = ds.views[2]
    full = pts_culling(view, PC).cpu().numpy()
    ids = pts_culling(view, PC, view_time=0.5).cpu().numpy()
    tf = np.float32(0.5)
    keep = (pres[full, 0] <= tf) & (tf <= pres[full, 1])
    assert np.array_equal(ids, full[keep])
