"""One process per rank on ONE B200 (the multi-process distributed path).

k = 2 and k = 3 processes (tests/mp_rank_worker.py) each build their row block
of the reference's golden matrices (tests/golden/dist.npz), connect through the
library's CUDA-IPC transport (send slots pulled by copy-engine peer copies,
stream-ordered flags -- no kernel waits on another rank, so ranks sharing one
GPU cannot deadlock), and run y = A x with three dots plus the fused golden
cases f1/f2 (shift/vshift, AXPBY, chain, dots) four times each: eager, CUDA
graph capture, graph replay, eager with SMs reserved for the pack.  Every repetition must reproduce the reference's
own dist_spmv (proj/src/partition.hpp:423-549) bit for bit in y and z, and its
dots within 1e-12 * (1 + sum |x||y|) (the reference sums its dots per worker).
"""
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_ranks(k, cases, transport="ipc", timeout=600):
    out = tempfile.mkdtemp(prefix="sk_mp_")
    port = _free_port()
    procs = []
    for r in range(k):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(k), LOCAL_RANK=str(r), LOCAL_WORLD_SIZE=str(k),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "mp_rank_worker.py"), out,
                                       ",".join(cases), transport], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=timeout)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for r, (p, log) in enumerate(zip(procs, logs)):
        assert p.returncode == 0, f"rank {r} failed:\n{log[-4000:]}"
    return [np.load(os.path.join(out, f"rank{r}.npz")) for r in range(k)]


def _ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("k,transport", [(2, "ipc"), (3, "ipc"), (2, "nccl"), (3, "nccl")])
def test_multiprocess_matches_reference_golden(golden, k, transport):
    """IPC runs with any number of GPUs (ranks share them); NCCL needs one GPU per rank."""
    from fused_cases import FUSED
    if transport == "nccl" and _ngpus() < k:
        pytest.skip(f"NCCL transport needs {k} GPUs, {_ngpus()} visible")
    g = golden("dist.npz")
    cases = sorted({"|".join(key.split("|")[:5]) for key in g.files
                    if "|crs|" not in key and key.split("|")[1] == str(k)})
    assert cases
    res = _run_ranks(k, cases, transport)
    w = 2
    for key in cases:
        off = g[key + "|row_offset"]
        n = int(off[-1])
        runs = [("plain", key, g[key + "|x"])] + [(f, f"{key}|{f}", g[f"{key}|{f}|x"]) for f, _, _ in FUSED]
        for fname, gk, xv in runs:
            for rep in range(4):
                y = np.concatenate([res[r][f"{key}|{fname}|{rep}|y"] for r in range(k)])
                dots = res[0][f"{key}|{fname}|{rep}|dot"]
                assert y.shape == (n, w)
                assert np.array_equal(y, g[gk + "|y"]), (key, fname, rep)   # bitwise, like the reference
                for r in range(1, k):                                      # every rank holds the same dots
                    assert np.array_equal(res[r][f"{key}|{fname}|{rep}|dot"], dots)
                sc = np.concatenate([np.sum(y ** 2, 0), np.sum(np.abs(xv * y), 0), np.sum(xv ** 2, 0)])
                if fname == "plain":
                    want = g[gk + "|dot"]
                    assert np.all(np.abs(dots - want) <= 1e-12 * (1 + sc)), (key, rep)
                else:
                    flags = dict((f, fl) for f, fl, _ in FUSED)[fname]
                    z = np.concatenate([res[r][f"{key}|{fname}|{rep}|z"] for r in range(k)])
                    assert np.array_equal(z, g[gk + "|z"]), (key, fname, rep)
                    want = g[gk + "|dot"]
                    for s in range(3):
                        if flags & (8 << s):  # DOT_YY << s
                            part = slice(s * w, (s + 1) * w)
                            assert np.all(np.abs(dots[part] - want[part]) <= 1e-12 * (1 + sc[part])), (key, fname)
                # graph replays repeat the eager result bit for bit (rep 3 runs a smaller
                # sweep grid, so its dot partials -- not y or z -- may differ in the last bits)
                if rep < 3:
                    assert np.array_equal(dots, res[0][f"{key}|{fname}|0|dot"])
        # halo bytes: the reference's count (minus its dot allreduce) per step, 12 steps;
        # the dot exchange adds 2(k-1) * 3w doubles per rank and step
        halo = int(g[key + "|comm"][0]) - 2 * (k - 1) * 3 * w * 8
        total = sum(int(res[r][f"{key}|stats"][0]) for r in range(k))
        assert total == 12 * halo + 12 * k * 2 * (k - 1) * 3 * w * 8, key
