"""bench.py contract checks that run without a GPU: the work model of
SURVEY.md 8(d) and the reference arm (``--impl reference``), which times the
reference algorithm on host cores and must print one JSON line the driver can
parse (impl, metric, unit, cpu_baseline, e2e with zero copied bytes)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_work_model_matches_survey():
    f, b = bench.work_per_matrix(4, "fwd")
    assert b == 144 and f == pytest.approx(8 / 3 * 64 + (6 * 4 + 24) * 4 * 3)
    f, b = bench.work_per_matrix(16, "fwdbwd")
    assert b == 4 * (2 * 256 + 16) + 4 * (3 * 256 + 32)
    assert f == pytest.approx(8 / 3 * 4096 + (6 * 16 + 24) * 16 * 15 + 6 * 4096 + 22 * 256)
    f, b = bench.work_per_matrix(8, "val")
    assert b == 4 * (64 + 8)
    bound, frac, flops, nbytes = bench.roofline(4, "fwd", 1 << 22, 0.268e-3, 6551.4e9)
    assert bound == "hbm" and nbytes == 144 * (1 << 22) and 0.3 < frac < 0.4


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "oracle")), reason="needs oracle/")
def test_reference_arm_prints_one_parseable_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == bench.METRIC and line["unit"] == bench.UNIT
    assert line["higher_is_better"] is True and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["n"] == bench.HEADLINE["n"]
