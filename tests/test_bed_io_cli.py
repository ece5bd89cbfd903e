"""BED1 I/O pinned to bytes written by the reference's
own write_batch (tests/golden/make_bed1.py), its error behaviour
(core.py:346-394), and the CLI exit codes of the reference harness
(cli.py:175-195).  CPU only; the GPU solve/gen/bench commands are in
tests/test_gpu_cli.py."""

import io
import os
import struct

import numpy as np
import pytest

import paper_2207_04228_b200 as bed
from paper_2207_04228_b200 import cli

HERE = os.path.join(os.path.dirname(__file__), "golden")


def test_reads_reference_bytes_bit_exact():
    ref = np.load(os.path.join(HERE, "ref_batch.npy"))
    m = bed.read_matrix(os.path.join(HERE, "ref_batch.bed"))
    np.testing.assert_array_equal(m.data, ref)
    assert np.signbit(m.data[0, 0, 0])  # -0.0 survives


def test_writes_reference_bytes():
    ref = np.load(os.path.join(HERE, "ref_batch.npy"))
    buf = io.BytesIO()
    bed.write_batch(bed.BatchedMatrix(ref), buf)
    with open(os.path.join(HERE, "ref_batch.bed"), "rb") as f:
        assert buf.getvalue() == f.read()


def test_symmetric_round_trip_and_shape_gate(tmp_path):
    a = np.random.default_rng(1).standard_normal((5, 6, 6))
    p = tmp_path / "a.bed"
    bed.write_batch(bed.BatchedSymmetric(a), p)
    np.testing.assert_array_equal(bed.read_batch(p).data, a)
    bed.write_batch(bed.BatchedMatrix(np.zeros((1, 2, 3))), p)
    with pytest.raises(bed.DimMismatch):
        bed.read_batch(p)


def test_format_errors():
    with pytest.raises(bed.BadMagic):
        bed.read_matrix(io.BytesIO(b"XXXX" + bytes(16)))
    with pytest.raises(bed.BadMagic):  # unsupported version
        bed.read_matrix(io.BytesIO(b"BED1" + struct.pack("<4I", 2, 1, 1, 1) + bytes(8)))
    with pytest.raises(bed.TruncatedPayload):
        bed.read_matrix(io.BytesIO(b"BED1" + struct.pack("<2I", 1, 1)))
    with pytest.raises(bed.TruncatedPayload):
        bed.read_matrix(io.BytesIO(b"BED1" + struct.pack("<4I", 1, 2, 2, 2) + bytes(8)))
    with pytest.raises(bed.DimMismatch):
        bed.read_matrix(io.BytesIO(b"BED1" + struct.pack("<4I", 1, 0, 2, 2)))


def test_cli_exit_codes(tmp_path):
    assert cli.main(["solve", str(tmp_path / "missing.bed"), "--out", str(tmp_path / "o")]) == cli.EXIT_IO
    bad = tmp_path / "bad.bed"
    bad.write_bytes(b"NOPE")
    assert cli.main(["solve", str(bad), "--out", str(tmp_path / "o")]) == cli.EXIT_IO
    assert cli.main(["gen", "--dims", "4,8", "--batches", "2", "--out", str(tmp_path / "g.bed")]) == cli.EXIT_USAGE
    with pytest.raises(SystemExit) as e:
        cli.main(["bench", "--dims", "x"])
    assert e.value.code == 2
