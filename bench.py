#!/usr/bin/env python
"""Benchmark of the B200 SELL-C-sigma SpMMV hot path (BASELINE.json metric:
"SELL-C-sigma SpMMV GFLOP/s and HBM GB/s vs roofline at 1/2/4/8 B200").

Workload (BASELINE.json configs[4], the north-star target): 3-D 7-point
Laplacian on a 400^3 grid (64M rows, 447,040,000 nonzeros), SELL-32-256,
row-major block vector of width 8, double, flags 0 (y = A x).  At N GPUs the
rows are distributed BY_ROWS (400/N z-planes per GPU, strong scaling) with an
NCCL halo exchange overlapped with the local sweep.

    python bench.py                      # N=1, defaults
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference     # the reference CPU library on this host

One JSON line on rank 0.  "value" = aggregate GFLOP/s (2*nnz*w per step, the
reference's flop convention, proj/tools/spmvbench.cpp:257) with inputs resident
in HBM, timed with CUDA events on the library stream, max over ranks.  "e2e" =
the same metric through the C ABI with host buffers (copy_in of x from pinned
memory, sellkit_spmv, copy_out of y) inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SELL-C-sigma SpMMV GFLOP/s and HBM GB/s vs roofline at 1/2/4/8 B200"
UNIT = "GFLOP/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=400, help="grid edge of the 3-D 7-point stencil")
    p.add_argument("--width", type=int, default=8)
    p.add_argument("--chunk", type=int, default=32)
    p.add_argument("--sigma", type=int, default=256)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-planes", type=int, default=40, help="z-planes of the bounded CPU sample")
    p.add_argument("--cpu-reps", type=int, default=10)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def stencil_nnz(n: int) -> int:
    return 7 * n ** 3 - 6 * n ** 2


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks --

class ClockSampler:
    """nvidia-smi samples DURING the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-i", str(self.device),
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ CPU reference --

def cpu_reference(planes: int, n: int, width: int, chunk: int, sigma: int, reps: int, warmup: int):
    """The reference's own CPU library (oracle/_ref, built from /root/reference by
    oracle/Makefile.ref) on a bounded sample: a 3-D 7-point box of n x n x planes
    rows (the per-row structure of the workload), all host cores.  Falls back to
    the oracle port (single thread) when the reference build is absent."""
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    os.environ.setdefault("SELLKIT_NUM_WORKERS", str(cores))
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    from oracle.oracle import REF_LIB_PATH, Oracle, hash_block, stencil_box
    rowptr, col, val = stencil_box(n, n, planes)
    nrows = len(rowptr) - 1
    nnz = int(rowptr[-1])
    xv = hash_block(nrows, width, 42)
    sample = f"3-D 7-pt box {n}x{n}x{planes} ({nrows} rows, {nnz} nnz), SELL-{chunk}-{sigma}, w={width}"
    flops = 2.0 * nnz * width
    times = []
    if os.path.exists(REF_LIB_PATH):
        from paper_1507_08101_b200 import sellkit
        ref = sellkit.Sellkit(REF_LIB_PATH, ext=False)
        ref.call("sellkit_set_num_workers", int(os.environ["SELLKIT_NUM_WORKERS"]))
        A = ref.crs(rowptr, col, val).build(chunk, sigma)
        x = ref.densemat_from(xv)
        y = ref.densemat(nrows, width)
        for i in range(warmup + reps):
            t0 = time.perf_counter()
            ref.spmv(y, A, x)
            if i >= warmup:
                times.append(time.perf_counter() - t0)
        kind, used = "reference", int(os.environ["OMP_NUM_THREADS"])
    else:
        orc = Oracle()
        A = orc.build(rowptr, col, val, chunk, sigma)
        for i in range(1 + max(1, reps // 3)):
            t0 = time.perf_counter()
            orc.spmv(A, xv)
            if i >= 1:
                times.append(time.perf_counter() - t0)
        kind, used = "port", 1
    t = float(np.median(times))
    return {"value": flops / t / 1e9, "unit": UNIT, "cores": used, "kind": kind, "sample": sample,
            "ms_per_step": t * 1e3, "steps": len(times)}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    cb = cpu_reference(args.cpu_planes, args.n, args.width, args.chunk, args.sigma, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": cb["steps"], "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"3-D 7-pt stencil {args.n}^3 SELL-{args.chunk}-{args.sigma} SpMMV w={args.width} "
                               f"(reference CPU on a bounded sample)", "sample": cb["sample"]},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours --

def run_ours(args, rank, world, local_rank):
    import torch
    from paper_1507_08101_b200 import sellkit

    torch.cuda.set_device(local_rank)
    sk = sellkit.load()
    n, w = args.n, args.width
    N = n ** 3
    nnz_total = stencil_nnz(n)
    if world > 1 or os.environ.get("SELLKIT_BENCH_RANKCTX") == "1":
        # one process per GPU: rank context (NCCL halo exchange); SELLKIT_BENCH_RANKCTX=1
        # exercises the same path at world size 1
        from paper_1507_08101_b200 import dist as skdist
        job = skdist.bench_setup(sk, n, w, args.chunk, args.sigma, rank, world)
    else:
        job = None

    stream = torch.cuda.ExternalStream(sk.stream())
    if job is None:
        crs = sk.crs_stencil(7, n)
        A = crs.build(args.chunk, args.sigma)
        del crs
        rows_local = N
        x = sk.densemat(N, w)
        x.fill_hash(42)
        y = sk.densemat(N, w)

        def step():
            sk.spmv(y, A, x)
        launches_per_step = 1
        nnz_local = nnz_total
    else:
        step = job.step
        launches_per_step = job.launches_per_step
        rows_local = job.rows_local
        nnz_local = job.nnz_local

    sk.set_sync(False)
    for _ in range(args.warmup):
        step()
    sk.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()

    clocks = ClockSampler(torch.cuda.current_device())
    if rank == 0:
        clocks.start()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with torch.cuda.stream(stream):
        evs[0].record(stream)
        for i in range(args.steps):
            step()
            evs[i + 1].record(stream)
    sk.synchronize()
    torch.cuda.synchronize()
    clk = clocks.stop() if rank == 0 else None
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    total_ms = evs[0].elapsed_time(evs[-1])
    sk.set_sync(True)

    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    flops_step = 2.0 * nnz_total * w
    value = flops_step / (ms_per_step * 1e-3) / 1e9

    # algorithmic bytes: 12 B/nnz + x read + y write, per GPU
    halo_bytes = job.halo_bytes if job is not None else 0
    alg_bytes = 12.0 * nnz_local + 8.0 * w * rows_local * 2 + halo_bytes
    kernel_ms = float(np.mean(per_step)) if job is None else job.kernel_ms(per_step)
    peak, peak_kind = measured_peaks()
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f)
        key = f"n{n}_w{w}_C{args.chunk}_s{args.sigma}_g{world}"
        traffic = tr.get(key)

    # -------- e2e through the C ABI with host buffers (rank-local rows)
    e2e = None
    if not args.no_e2e:
        if job is None:
            xh = torch.empty((N, w), dtype=torch.float64, pin_memory=True)
            yh = torch.empty((N, w), dtype=torch.float64, pin_memory=True)
            ptr_x, ptr_y = xh.data_ptr(), yh.data_ptr()
            nel = N * w
            sk.call("sellkit_densemat_copy_out", x.h, sellkit.vp(ptr_x), nel)  # the step's input lives on the host
            # sellkit_spmv straight on host buffers (view_plain of pinned memory): the library
            # streams x in and y out by row blocks, overlapping both copy engines with the sweep
            xv_h = sk.view_plain(ptr_x, nel, N, w, w, keep=xh)
            yv_h = sk.view_plain(ptr_y, nel, N, w, w, keep=yh)

            def e2e_step():
                sk.spmv(yv_h, A, xv_h)
            h2d = d2h = nel * 8
        else:
            e2e_step, h2d, d2h = job.e2e_step, job.h2d_bytes, job.d2h_bytes
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        if job is not None and job.e2e_flush is not None:
            job.e2e_flush()
        e1.record(stream)
        torch.cuda.synchronize()
        sk.set_sync(True)
        te = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], dtype=torch.float64, device="cuda")
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": flops_step / (float(te.item()) * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": float(te.item()), "steps": args.e2e_steps,
               "path": ("sellkit_spmv on view_plain host buffers (pinned), streamed H2D/sweep/D2H"
                        if job is None else "per rank: H2D x, sellkit_ext_rank_spmv, D2H y; consecutive steps "
                        "overlap the upload with the previous download")}

    if rank != 0:
        return
    cb = None
    if not args.no_cpu_baseline:
        cb = cpu_reference(args.cpu_planes, n, w, args.chunk, args.sigma, args.cpu_reps, 1)
        cb = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"3-D 7-pt Laplacian {n}^3 ({N} rows, {nnz_total} nnz), SELL-{args.chunk}-{args.sigma}, "
                               f"row-major block width {w}, y = A x",
                   "rows": N, "nnz": nnz_total, "block_width": w, "chunk_height": args.chunk, "sigma": args.sigma,
                   "parallelism": f"rows{world}", "l2": "inputs (13.6 GB) >> 126 MB L2, no flush needed",
                   "hbm_gbs_aggregate": alg_bytes * world / (ms_per_step * 1e-3) / 1e9},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind, "alg_bytes_per_launch": alg_bytes,
                     "kernel_ms": kernel_ms},
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "cpu_baseline": cb,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
