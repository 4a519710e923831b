"""The driver's bench command on the GPU, small: the N = 1 line and the N = 2 rank path
(torch.distributed.run, IPC halo transport, CUDA-graph steps) with both ranks sharing the one
GPU of the test box (SELLKIT_BENCH_SHARE_GPUS=1: a protocol run, marked gpus_shared)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env=None, timeout=900):
    e = dict(os.environ)
    e.update(env or {})
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def _check_line(line, n_gpus):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert key in line, key
    assert line["n_gpus"] == n_gpus and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0


def test_bench_one_gpu_small():
    line = _bench("--n", "96", "--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    _check_line(line, 1)
    assert line["construction"]["spmv_units_build"] > 0


def test_bench_two_ranks_sharing_the_gpu():
    line = _bench("--gpus", "2", "--n", "96", "--steps", "5", "--warmup", "3", "--no-cpu-baseline",
                  env={"SELLKIT_BENCH_SHARE_GPUS": "1"})
    _check_line(line, 2)
    assert line["config"]["gpus_shared"] is True
    assert line["config"]["halo_transport"] == "ipc"
