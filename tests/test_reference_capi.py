"""The reference's OWN C-ABI test suite (proj/tests/unit_capi.cpp, plus the C99 header
check proj/tests/c_api_compile.c), compiled unmodified by oracle/Makefile.ref against a
doctest stand-in (tests/doctest_shim/doctest.h):

* against the reference library itself (CPU): validates the stand-in -- all 11 cases pass;
* against THIS library's include/sellkit.h and libsellkit_b200.so (GPU): the drop-in
  boundary proof.  The two task-pool cases are excluded: the host-CPU task pool is out
  of scope and its entry points return SELLKIT_ERR_UNSUPPORTED
  (tests/test_capi_cpu.py checks that contract).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "unit_capi_ref")
B200_BIN = os.path.join(ROOT, "oracle", "_ref", "unit_capi_b200")
OUT_OF_SCOPE = ["task dependencies through the C API", "task pool through the C API"]


def _run(path, *args):
    if not os.path.exists(path):
        pytest.skip(f"{os.path.relpath(path, ROOT)} not built (python -m oracle.build)")
    r = subprocess.run([path, *args], capture_output=True, text=True, timeout=600, cwd="/tmp")
    return r.returncode, r.stdout + r.stderr


def test_reference_suite_on_reference_library():
    rc, out = _run(REF_BIN)
    assert rc == 0, out
    assert "test cases: 11 run, 0 failed, 0 skipped" in out, out


@pytest.mark.gpu
def test_reference_suite_on_b200_library():
    rc, out = _run(B200_BIN, "-tce=" + ",".join(OUT_OF_SCOPE))
    assert rc == 0, out
    assert "test cases: 9 run, 0 failed, 2 skipped" in out, out
