"""Build the B200 library (and, for tests/bench only, the CPU oracle).

    python -m paper_1507_08101_b200.build            # product library only
    python -m paper_1507_08101_b200.build --all      # + oracle/liboracle.so + oracle/_ref (if /root/reference exists)
"""
from __future__ import annotations

import os
import subprocess
import sys

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


def build_oracle() -> None:
    """The CPU checker (test infrastructure, never linked by the product)."""
    _run(["make", "-f", "oracle/Makefile"])
    if os.path.isdir("/root/reference/proj"):
        _run(["make", f"-j{max(1, os.cpu_count() or 1)}", "-f", "oracle/Makefile.ref"])


if __name__ == "__main__":
    build_library()
    if "--all" in sys.argv:
        build_oracle()
