import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def cells():
    import numpy as np

    with np.load(os.path.join(GOLDEN, "cells.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def known():
    import numpy as np

    with np.load(os.path.join(GOLDEN, "known_answers.npz")) as z:
        return {k: z[k] for k in z.files}


def cell_names(cells_dict):
    return sorted({k.split("/")[0] for k in cells_dict if k.endswith("/a")})
