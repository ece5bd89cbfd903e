"""The CLI's GPU commands: gen -> solve round trip
through BED1 files, checked against the float64 oracle; bench CSV schema."""

import numpy as np
import pytest

import oracle
import parity as P
import paper_2207_04228_b200 as bed
from paper_2207_04228_b200 import cli

pytestmark = pytest.mark.gpu


def test_gen_solve_round_trip(tmp_path):
    src = tmp_path / "a.bed"
    assert cli.main(["gen", "--dims", "12", "--batches", "40", "--seed", "3", "--out", str(src)]) == 0
    a = bed.read_batch(src).data
    assert a.shape == (40, 12, 12)
    assert cli.main(["solve", str(src), "--out", str(tmp_path / "r"), "--tol", "3e-12"]) == 0
    lam = bed.read_matrix(tmp_path / "r.values.bed").data[:, :, 0]
    vec = bed.read_matrix(tmp_path / "r.vectors.bed").data
    o = oracle.forward(a)
    assert np.all(P.eig_err(lam, o.eigenvalues) <= P.EIG_TOL)
    assert np.all(P.recon_err(a, lam, vec) <= P.RECON_TOL)
    assert cli.main(["solve", str(src), "--out", str(tmp_path / "v"), "--no-vectors"]) == 0
    assert not (tmp_path / "v.vectors.bed").exists()


def test_solve_reports_invalid_input(tmp_path):
    a = np.stack([np.eye(4)] * 2)
    a[1, 0, 1] = 5.0  # asymmetric
    p = tmp_path / "bad.bed"
    bed.write_batch(bed.BatchedMatrix(a), p)
    assert cli.main(["solve", str(p), "--out", str(tmp_path / "o")]) == cli.EXIT_FAIL


def test_bench_csv(capsys):
    assert cli.main(["bench", "--dims", "4,16", "--batches", "64", "--reps", "2"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == cli.CSV_HEADER
    assert len(lines) == 3 and lines[1].startswith("4,64,full,")


def test_bench_csv_counters(capsys):
    assert cli.main(["bench", "--dims", "12", "--batches", "32", "--reps", "1"]) == 0
    row = capsys.readouterr().out.strip().splitlines()[1].split(",")
    mean_r, mean_k, rotations = float(row[5]), float(row[6]), int(row[7])
    assert 0 < mean_r < 10 and mean_k > 1 and rotations > 32 * 10
    assert row[8] == ""  # max_eig_err is a verify-run quantity (reference bench.py:71)


def test_verify_grid_passes(capsys):
    rc = cli.main(["verify", "--dims", "4,12,24", "--batches", "1,64", "--count", "128", "--csv"])
    out = capsys.readouterr().out.strip().splitlines()
    assert out[0] == "dim,batch,count,max_eig_err,max_recon,max_orth,max_single_dev,r_median,passed"
    assert len(out) == 7
    assert rc == cli.EXIT_OK, out
    for line in out[1:]:
        f = line.split(",")
        assert int(f[2]) >= 128 and float(f[3]) <= 1e-5 and f[-1] == "1"
        assert float(f[6]) == 0.0  # per-matrix deflation: batch and single solves agree exactly


def test_verify_table_and_failing_gate(capsys):
    assert cli.main(["verify", "--dims", "8", "--batches", "16", "--count", "16"]) == cli.EXIT_OK
    text = capsys.readouterr().out
    assert "eig_err" in text and "pass" in text
    # an impossible gate fails the cell and the exit status
    assert cli.main(["verify", "--dims", "8", "--batches", "16", "--count", "16", "--tol", "1e-30"]) == cli.EXIT_FAIL
