"""Process-level tests of the spmvbench driver (paper_1507_08101_b200/bin/spmvbench),
mirroring the reference's proj/tests/unit_cli.cpp and acceptance criterion 9
(byte-identical report against tests/golden/spmvbench_identity.txt, copied from
the reference's proj/tests/golden/)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1507_08101_b200", "bin", "spmvbench")
GOLDEN = os.path.join(ROOT, "tests", "golden", "spmvbench_identity.txt")

pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="spmvbench not built")


def run(args):
    p = subprocess.run([BIN] + args.split(), capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


# --- usage and I/O errors exit before any device work (CPU) ----------------
@pytest.mark.parametrize("args", ["-m identity:64 -f SELL-0-1", "-m identity:64 -f CRS",
                                  "-m identity:64 --unknown-flag", "", "-m identity:64 -w 1:2.75",
                                  "-m identity:64 -w 1:xyz --ranks 2", "-m identity:64 -n 0",
                                  "-m identity:64 -s fast", "-m identity:64 --mode eager", "-m"])
def test_usage_errors_exit_1(args):
    assert run(args)[0] == 1


def test_io_errors_exit_2():
    assert run("-m /nonexistent/matrix.mtx")[0] == 2
    assert run("-m /nonexistent/matrix.gcrs")[0] == 2


# --- runs (device) ---------------------------------------------------------
@pytest.mark.gpu
def test_golden_report_byte_identical():
    rc, out, _ = run("-m identity:1000 --fake-timer")
    assert rc == 0
    assert out == open(GOLDEN).read()


@pytest.mark.gpu
def test_format_and_weights():
    rc, out, _ = run("-m identity:64 -f SELL-32-1 --fake-timer -n 20")
    assert rc == 0 and "spmv (GF/s)" in out
    assert run("-m laplace:100 -f SELL-4-4 --ranks 2 -w 1:2.75 --fake-timer -n 15")[0] == 0


@pytest.mark.gpu
def test_few_iterations_print_na():
    rc, out, _ = run("-m identity:64 -n 5 --fake-timer")
    assert rc == 0 and "     n/a" in out


@pytest.mark.gpu
def test_nocomm_matches_default_on_one_rank():
    a = run("-m laplace:200 -f SELL-4-4 --fake-timer -n 12")
    b = run("-m laplace:200 -f SELL-4-4 -s nocomm --fake-timer -n 12")
    assert a[0] == 0 and b[0] == 0 and a[1] == b[1]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["nooverlap", "naive", "task"])
def test_modes(mode):
    rc, out, _ = run(f"-m laplace:300 -f SELL-4-4 --ranks 2 --mode {mode} --fake-timer -n 12")
    assert rc == 0 and "spmv (GF/s) |    12 |" in out


@pytest.mark.gpu
def test_verbose_rank_warning_and_comm_stats():
    rc, _, err = run("-m identity:64 -v --ranks 5 --fake-timer -n 12")
    assert rc == 0
    assert "[GHOST] PERFWARNING: The number of MPI ranks (5)" in err and "Suggested number:" in err
    assert "communication:" in err


@pytest.mark.gpu
def test_width_feeds_flop_accounting():
    assert "2.00e-03" in run("-m identity:1000 --fake-timer -n 20")[1]
    assert "8.00e-03" in run("-m identity:1000 --width 4 --fake-timer -n 20")[1]


@pytest.mark.gpu
def test_matrix_files(tmp_path):
    mm = tmp_path / "t.mtx"
    mm.write_text("%%MatrixMarket matrix coordinate real symmetric\n4 4 5\n1 1 2\n2 1 -1\n2 2 2\n3 3 2\n4 4 2\n")
    rc, out, _ = run(f"-m {mm} -f SELL-2-2 --fake-timer -n 12")
    assert rc == 0 and "spmv (GF/s) |    12 |" in out
