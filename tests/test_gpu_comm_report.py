"""Locality vs random all-to-all accounting at a small configuration
(paper_2512_20017_b200.comm_report; the full C4/C5 runs are committed under
profiles/)."""

import pytest

from paper_2512_20017_b200 import comm_report

pytestmark = pytest.mark.gpu


def test_comm_report_tiny(cuda):
    res = comm_report.run(comm_report.CONFIGS["tiny"], [2, 4], epochs=1, log=lambda *_: None)
    for n in ("2", "4"):
        row = res["per_gpus"][n]
        assert row["steps"] == 32 // 8
        loc, rnd = row["fwd_points_per_step"]["locality"], row["fwd_points_per_step"]["random"]
        assert 0 <= loc < rnd
        assert row["reduction_pct"] == pytest.approx(100.0 * (1.0 - loc / rnd))
        assert row["fwd_bytes_per_step"]["locality"] == loc * comm_report.SP_BYTES  # 48-byte row + 4-byte id
