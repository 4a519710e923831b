"""Build the B200 library in-tree (paper_1507_08101_b200/lib/libsellkit_b200.so).

    python -m paper_1507_08101_b200.build

The CPU checkers are test infrastructure and build separately (python -m oracle.build).
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "lib", "libsellkit_b200.so")


def _run(cmd, cwd=ROOT):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, cwd=cwd, check=True)


def build_library(jobs: int = 0) -> str:
    jobs = jobs or max(1, os.cpu_count() or 1)
    _run(["make", f"-j{jobs}", "-C", os.path.join(HERE, "csrc")])
    if not os.path.exists(LIB):
        raise RuntimeError(f"build did not produce {LIB}")
    return LIB


if __name__ == "__main__":
    build_library()
