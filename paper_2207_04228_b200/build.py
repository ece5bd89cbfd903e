"""Build libbed200.so in-tree (nvcc, sm_100a) via csrc/Makefile."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")


def build(jobs: int | None = None, verbose: bool = False) -> str:
    jobs = jobs or max(1, os.cpu_count() or 1)
    cmd = ["make", "-C", CSRC, f"-j{jobs}"]
    if not verbose:
        cmd.append("-s")
    subprocess.run(cmd, check=True)
    from ._native import LIB_PATH

    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"build finished but {LIB_PATH} is missing")
    return LIB_PATH


if __name__ == "__main__":
    print(build(verbose=True))
