"""bench.py contract checks that run without a GPU: the reference arm (CPU
oracle) prints one JSON line with the required keys, and the weak-scaling
configuration helper keeps per-rank work fixed."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"


def test_weak_scaled_config():
    import bench

    c = bench.weak_scaled(bench.CONFIGS["c2"], 4)
    assert c["n_points"] == 4 * bench.CONFIGS["c2"]["n_points"]
    assert c["grid"] == (1, 4) and c["n_views"] == 32 and c["batch"] == bench.CONFIGS["c2"]["batch"]


def test_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks
    (torch.distributed.run on 127.0.0.1) and rank 0 prints the only line."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--gpus", "2", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=900,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    assert d["config"]["global_batch"] == 2 and d["config"]["parallelism"] == "points+images x2"


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--gpus", "2", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_roofline_model():
    """roofline.py: the frozen per-stage compulsory bytes add up to the step,
    and the binding bound is the larger fraction."""
    from paper_2512_20017_b200 import roofline as rl

    c = {"S": 1_000_000, "V": 4_000_000, "Vp": 1_000_000, "I": 8_500_000, "Np": 4 * 1920 * 1080,
         "nb": 4 * 8160, "gsp_clear": True}
    parts = {s: rl.stage_bytes(s, c) for s in ("cull", "project", "bin", "raster_fwd", "raster_bwd",
                                                "project_bwd_adam")}
    assert parts["bin"] == 20 * c["V"] + 20 * c["I"] + 8 * c["nb"]
    assert parts["project_bwd_adam"] == 6 * 240 * c["S"] + 4 * c["S"] + 36 * c["V"]
    assert rl.step_bytes(c) == sum(parts.values())
    assert rl.survey_step_bytes(c) > 0
    h = rl.hbm(parts["raster_bwd"], 1.9, 6539.5)
    i = rl.issue(1.6e9, 1.9, 1965.0)
    assert rl.binding(h, i) == "issue" and rl.binding(rl.hbm(1.5e9, 0.3, 6539.5), None) == "hbm"
    assert rl.binding(h, None) is None  # issue rate not captured and far from the HBM bound: not called
