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
