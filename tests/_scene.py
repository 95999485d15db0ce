"""Shared test fixtures: small scenes in the kernels' layout, oracle pipelines."""

from __future__ import annotations

import numpy as np

from paper_2512_20017_b200 import scenes
from paper_2512_20017_b200.culling import batch_planes, patch_edges  # noqa: F401

C1 = dict(seed=0, n_points=10_000, grid=(2, 2), n_views=8, altitude=50.0, image_size=(128, 128))


def host_group_layout(cloud: scenes.PointCloud, G: int):
    """Z-order sort + groups on the host (oracle restatement of
    visibility.py:113-134), used to build inputs without a GPU."""
    from oracle import py_oracle

    return py_oracle.zorder_layout(cloud.positions, G)


def c1_setup(G: int = 256, **over):
    cfg = dict(C1, **over)
    ds = scenes.generate_aerial_scene(cfg["seed"], cfg["n_points"], cfg["grid"], cfg["n_views"], cfg["altitude"],
                                      cfg["image_size"])
    perm, gb, aabb = host_group_layout(ds.cloud, G)
    sorted_cloud = scenes.PointCloud(ds.cloud.positions[perm])
    spacing = scenes.mean_spacing(cfg["altitude"], cfg["grid"], cfg["n_points"])
    params = scenes.init_gaussians(sorted_cloud, cfg["seed"], spacing)
    W, H = cfg["image_size"]
    gt = scenes.synthetic_gt(cfg["seed"], cfg["n_views"], W, H)
    return ds, params, gb, aabb, gt


def oracle_view_pipeline(params, gb, aabb, view, cam_bytes, gt_img, sh_degree=3, model="3dgs", bg=(0.0, 0.0, 0.0)):
    """Oracle forward + backward of one view; returns dict of intermediates."""
    from oracle import py_oracle

    planes = batch_planes([view], 1)
    pos = params[0, :, :3]
    mask = py_oracle.visibility_mask(pos, gb, aabb, planes, 1)
    idx = np.flatnonzero(mask & 1).astype(np.int64)
    sp = py_oracle.project(params, idx, cam_bytes, sh_degree, model=model)
    img, T, nc, lists, ranges = py_oracle.render(sp, view.width, view.height, bg=bg, want_lists=True, model=model)
    loss, gimg = py_oracle.l1_loss(img, gt_img)
    gsp = py_oracle.render_bwd(sp, view.width, view.height, T, nc, gimg, bg=bg, model=model)
    gparams = py_oracle.project_bwd(params, idx, cam_bytes, sh_degree, gsp, model=model)
    return dict(mask=mask, idx=idx, sp=sp, img=img, T=T, nc=nc, lists=lists, ranges=ranges, loss=loss, gimg=gimg,
                gsp=gsp, gparams=gparams)
