"""Writes tests/golden/ref_batch.bed with the REFERENCE package's own
write_batch (/root/reference/pkg/src/batchedeig/core.py:333-343), so the
BED1 reader/writer of this repo is pinned to the reference bytes.  Run in the
build container (the reference is not on the GPU box):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bed1.py
"""
import os

import numpy as np
from batchedeig.core import BatchedMatrix, write_batch

rng = np.random.default_rng(20261017)
data = rng.standard_normal((3, 4, 5))
data[0, 0, 0] = -0.0
data[1, 2, 3] = 1e-300
data[2, 3, 4] = np.finfo(np.float64).max
out = os.path.join(os.path.dirname(__file__), "ref_batch.bed")
write_batch(BatchedMatrix(data), out)
np.save(os.path.join(os.path.dirname(__file__), "ref_batch.npy"), data)
print("wrote", out)
