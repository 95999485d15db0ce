"""Frozen roofline model of the training step.

Algorithmic (compulsory) bytes per launch of every stage: each kernel reads
its distinct inputs once and writes its outputs once; nothing it could keep
on chip or in L2 is counted twice.  Counts come from one step:

  S    points of the rank's shard            V    splat rows (visible (point, view) pairs)
  Vp   visible points (>= 1 batch view)      I    tile instances
  Np   rendered pixels (slots x H x W)       nb   (slot, tile) buckets

Per model (include/splat_b200.h): parameter row 240 B (59 live f32 + pad,
plane-major float4), SP row 48 B (3DGS) / 96 B (2DGS), G_SP wire 36 B /
60 B, raster gather per instance 36 B / 64 B (the fields of the SP row the
blend reads) + 4 B list entry.

| stage            | bytes                                                        |
|------------------|--------------------------------------------------------------|
| cull             | 16 S (plane-0 float4) + 4 S (mask)                           |
| project          | 240 Vp + 4 S + SProw V  (+ G_SP clear 48 V when fused)       |
| bin              | 20 V (centre, depth, extents) + 8 I (key write) + 8 I (key   |
|                  | read) + 4 I (list write) + 8 nb (ranges)                     |
| raster_fwd       | (4 + gather) I + 23 Np (rgb 12, T 4, n 4 written, gt 3 read) |
| raster_bwd       | (4 + gather) I + 23 Np (image, T, n, gt read) + G_SP V       |
| raster (fused)   | (4 + gather) I + 23 Np (rgb, T, n written, gt read) + G_SP V |
|                  | (K3 + L + K4 in one kernel: the list and the pixel state are |
|                  | read once)                                                   |
| project_bwd_adam | 6 x 240 S (p, m, v read + write) + 4 S + G_SP V              |
|                  | (selective Adam: 6 x 240 Vp + 4 S + G_SP V)                  |

The SURVEY's own formula (§8(d), `survey_step_bytes`) is kept beside it for
comparison; it assumes 4(K-3) + 44 B per projected row and 44 B per
instance for the sort.  Peaks: the measured HBM copy bandwidth
(MEASURED_PEAKS.json `hbm_gbs`), the warp-instruction issue rate
148 SMs x 4 schedulers x SM clock.  The raster kernels are issue-bound, the
per-point kernels HBM-bound: `binding()` names whichever fraction is higher.
"""

from __future__ import annotations

import json
import os

N_SM = 148
SCHEDULERS = 4
PARAM_ROW = 240

MODEL = {
    # sp row, G_SP wire, raster gather per instance (without the 4 B list entry)
    "3dgs": dict(sp=48, gsp=36, gather=36),
    "2dgs": dict(sp=96, gsp=60, gather=64),
}


def stage_bytes(stage: str, c: dict, model: str = "3dgs") -> int | None:
    """Compulsory bytes of one launch of `stage` given step counts `c`
    (keys S, V, Vp, I, Np, nb, gsp_clear, selective)."""
    m = MODEL[model]
    S, V, I, Np = c["S"], c["V"], c["I"], c["Np"]
    if stage == "cull":
        return 16 * S + 4 * S
    if stage == "project":
        return PARAM_ROW * c.get("Vp", S) + 4 * S + m["sp"] * V + (48 * V if c.get("gsp_clear") else 0)
    if stage == "bin":
        return 20 * V + 8 * I + 8 * I + 4 * I + 8 * c.get("nb", 0)
    if stage == "raster_fwd":
        return (4 + m["gather"]) * I + 23 * Np
    if stage == "raster_bwd":
        return (4 + m["gather"]) * I + 23 * Np + m["gsp"] * V
    if stage == "raster":  # fused forward + loss + backward (bs_raster_fwd_bwd)
        return (4 + m["gather"]) * I + 23 * Np + m["gsp"] * V
    if stage == "project_bwd_adam":  # selective Adam: only the visible points' rows move
        n_upd = c.get("Vp", S) if c.get("selective") else S
        return 6 * PARAM_ROW * n_upd + 4 * S + m["gsp"] * V
    return None


def step_bytes(c: dict, model: str = "3dgs", stages=("cull", "project", "bin", "raster_fwd", "raster_bwd",
                                                      "project_bwd_adam")) -> int:
    return int(sum(stage_bytes(s, c, model) or 0 for s in stages))


def survey_step_bytes(c: dict, K: int = 59, E: int = 11, Eg: int = 9) -> int:
    """SURVEY.md §8(d) frozen formula for one step (all views of the batch)."""
    S, V, I, Np = c["S"], c["V"], c["I"], c["Np"]
    Vloc = V
    cull = 12 * S
    project = 4 * (K - 3) * Vloc + 4 * E * Vloc
    binning = 12 * I + 24 * I + 8 * I
    fwd = 40 * I + 20 * Np
    loss = 36 * Np
    bwd = 40 * I + 20 * Np + 4 * Eg * V
    pbwd = 4 * K * Vloc + 4 * Eg * Vloc + 4 * K * Vloc
    adam = 28 * K * S
    return int(cull + project + binning + fwd + loss + bwd + pbwd + adam)


def hbm(bytes_: float, ms: float, peak_gbs: float) -> dict:
    ach = bytes_ / (ms / 1000.0) / 1e9 if ms and bytes_ else None
    return {"bound": "hbm", "achieved": ach, "peak": peak_gbs, "unit": "GB/s",
            "frac": (ach / peak_gbs) if ach else None, "bytes": int(bytes_) if bytes_ else None}


def issue(warp_instructions: float | None, ms: float, sm_mhz: float | None) -> dict | None:
    """Executed warp instructions of one launch over its duration against
    148 SMs x 4 schedulers x 1 issue/clock at the sampled SM clock."""
    if not warp_instructions or not ms or not sm_mhz:
        return None
    ach = warp_instructions / (ms / 1000.0) / 1e9
    peak = N_SM * SCHEDULERS * sm_mhz * 1e6 / 1e9
    return {"bound": "issue", "achieved": round(ach, 1), "peak": round(peak, 1), "unit": "G warp-instr/s",
            "frac": round(ach / peak, 4), "warp_instructions": warp_instructions}


def binding(h: dict | None, i: dict | None) -> str | None:
    """The bound a kernel actually sits against: the larger fraction (None when
    the issue rate was not captured for this workload and the HBM fraction is
    too low to call the kernel memory-bound)."""
    hf = (h or {}).get("frac") or 0.0
    if i is None or i.get("frac") is None:
        return "hbm" if hf >= 0.5 else None
    return "issue" if i["frac"] > hf else "hbm"


def peaks(root: str) -> tuple[float, str]:
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"
