"""bench.py --gpus 2 (self-launched ranks, both on cuda:0, over gloo (the driver runs
N > 1 under torchrun over NCCL on N GPUs; this checks the plumbing: weak
scaling, sharding, async placement, comm report, one JSON line)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("patches,exchange", [(1, "peer"), (1, "collective"), (2, "peer")])
def test_bench_two_ranks_gloo(cuda, patches, exchange):
    env = dict(os.environ, BS_DIST_BACKEND="gloo")
    # no torchrun wrapper: `--gpus 2` launches its own two ranks
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3", "--config",
           "c1", "--patches", str(patches), "--exchange", exchange]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["global_batch"] == 2
    assert d["config"]["patches_per_side"] == patches
    assert d["placement"]["async"] and d["placement"]["step_wait_ms"] is not None  # prefetched W used
    assert d["comm"]["fwd_bytes_per_step"] >= 0 and d["comm"]["random_fwd_bytes_per_step"] > 0
    assert d["comm"]["backend"] == "gloo" and d["comm"]["communicator_size"] == 2
    assert ("peer" in d["comm"]["exchange"]) == (exchange == "peer" and patches == 1)
    assert d["partition"]["built_on"] == "rank 0" and sum(d["partition"]["points_per_rank"]) == 2 * 10_000
    assert d["roofline"]["step_hbm"]["frac"] > 0
