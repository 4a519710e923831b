"""Build the CPU checkers (TEST INFRASTRUCTURE ONLY, never linked by the product):
oracle/liboracle.so + oracle/libfullsize.so, and oracle/_ref (the reference library
compiled from its own sources by oracle/Makefile.ref) when /root/reference exists.

    python -m oracle.build
"""
from __future__ import annotations

import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, cwd=ROOT, check=True)


def build_oracle() -> None:
    _run(["make", "-f", "oracle/Makefile"])
    if os.path.isdir("/root/reference/proj"):
        _run(["make", f"-j{max(1, os.cpu_count() or 1)}", "-f", "oracle/Makefile.ref"])


if __name__ == "__main__":
    build_oracle()
