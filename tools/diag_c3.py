"""Diagnostic: C3 (2DGS) view vs the oracle -- where do the images differ?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from paper_2512_20017_b200 import scenes
from paper_2512_20017_b200.culling import zorder_group
from paper_2512_20017_b200.trainer import SplatTrainer, camera_bytes
from _scene import oracle_view_pipeline

seed, n = 2, 2_000_000
ds = scenes.generate_aerial_scene(seed, n, (1, 1), 8, 50.0, (1920, 1080))
g = zorder_group(ds.cloud, G=2048)
params = scenes.init_gaussians(g.sorted_cloud, seed, scenes.mean_spacing(50.0, (1, 1), n))
gt = scenes.synthetic_gt(seed, 8, 1920, 1080)
gb, aabb = g.group_begin(), g.aabbs.reshape(-1, 6)
tr = SplatTrainer(params, gb, aabb, ds.views, gt=gt, model="2dgs")
batch = [2]
tr.step(batch)
torch.cuda.synchronize()
H, W = 1080, 1920
img = tr.last["image"][: H * W * 3].cpu().numpy().reshape(H, W, 3)
T = tr.last["final_T"][: H * W].cpu().numpy().reshape(H, W)
nc = tr.last["n_contrib"][: H * W].cpu().numpy().reshape(H, W)
sp = tr.last["sp"][: tr.last["n_rows"] * 24].cpu().numpy().reshape(-1, 24)
ref = oracle_view_pipeline(params, gb, aabb, ds.views[2], camera_bytes([ds.views[2]]), gt[2], model="2dgs")
d = np.abs(img - ref["img"]).max(axis=2)
bad = np.argwhere(d > 1e-4)
print("bad pixels", len(bad), "max", d.max())
print("n_contrib differs", int((nc != ref["nc"]).sum()), "T differs >1e-6", int((np.abs(T - ref["T"]) > 1e-6).sum()))
for (y, x) in bad[:8]:
    t = (y // 16) * ((W + 15) // 16) + x // 16
    a, b = ref["ranges"][t]
    lst = ref["lists"][a:b]
    print(f"pixel ({x},{y}) err {d[y,x]:.3e} nc gpu {nc[y,x]} ref {ref['nc'][y,x]} T gpu {T[y,x]:.6g} ref {ref['T'][y,x]:.6g}")
    rx, ry = (x // 8) * 8, (y // 4) * 4
    x0, x1, y0, y1 = rx + 0.5, rx + 7.5, ry + 0.5, ry + 3.5
    for i, r in enumerate(lst[: max(nc[y, x], ref["nc"][y, x]) + 2]):
        pass_ = True
        row = sp[r]
        cx, cy, hx, hy = row[22], row[23], row[16], row[17]
        reach = (abs(cx - min(max(cx, x0), x1)) <= hx * 1.0001 + 1e-3) and (abs(cy - min(max(cy, y0), y1)) <= hy * 1.0001 + 1e-3)
        inbox = abs(x + 0.5 - cx) <= hx and abs(y + 0.5 - cy) <= hy
        g2 = 2 * ((row[0] - x - 0.5) ** 2 + (row[1] - y - 0.5) ** 2)
        M = row[3:12].astype(np.float64).reshape(3, 3)
        hxv = M[0] - (x + 0.5) * M[2]
        hyv = M[1] - (y + 0.5) * M[2]
        z = np.cross(hxv, hyv)
        g3 = (z[0] ** 2 + z[1] ** 2) / z[2] ** 2 if z[2] != 0 else np.inf
        k = min(9.0, 2 * np.log(255 * row[2]))
        if not (min(g3, g2) <= k + 0.05) and not inbox:
            continue
        print(f"   #{i} row {r} o {row[2]:.3f} k {k:.3f} g3 {g3:.4f} g2 {g2:.4f} in {min(g3,g2) <= k} reach {reach} inbox {inbox} box ({cx:.2f},{cy:.2f})+-({hx:.2f},{hy:.2f})")
