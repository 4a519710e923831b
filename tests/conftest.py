import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no GPU in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle, LIB_PATH
    if not os.path.exists(LIB_PATH):
        import subprocess
        subprocess.run(["make", "-f", "oracle/Makefile"], cwd=ROOT, check=True)
    return Oracle()


@pytest.fixture(scope="session")
def sk():
    """The B200 library.  Loads the in-tree .so; fails loudly if it is missing."""
    from paper_1507_08101_b200 import sellkit
    return sellkit.load()


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name))
    return load


def storage_perm(A_layout):
    return A_layout["row_perm"]
