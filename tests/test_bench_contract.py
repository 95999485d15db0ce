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
