#!/usr/bin/env python
"""Benchmark of the B200 SELL-C-sigma SpMMV hot path (BASELINE.json metric:
"SELL-C-sigma SpMMV GFLOP/s and HBM GB/s vs roofline at 1/2/4/8 B200").

Workload (BASELINE.json configs[4], the north-star target): 3-D 7-point
Laplacian on a 400^3 grid (64M rows, 447,040,000 nonzeros), SELL-32-256,
row-major block vector of width 8, double, flags 0 (y = A x).  At N GPUs the
rows are distributed BY_ROWS (400/N z-planes per GPU, strong scaling), each
rank on its own GPU, with the halo exchange (CUDA-IPC slots pulled by copy
engines, or NCCL) overlapped with the local sweep.

    python bench.py                      # N=1, defaults
    python bench.py --gpus N             # starts N ranks itself (torch.distributed.run)
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference     # the reference CPU library on this host

One JSON line on rank 0.  "value" = aggregate GFLOP/s (2*nnz*w per step, the
reference's flop convention, proj/tools/spmvbench.cpp:257) with inputs resident
in HBM, timed with CUDA events on the library stream, max over ranks.  "e2e" =
the same metric through the C ABI with host buffers (x from pinned memory,
sellkit_spmv, y back to pinned memory) inside the timed region.  The reference
arm and "cpu_baseline" run the unmodified reference library (oracle/_ref, built
from /root/reference/proj by oracle/Makefile.ref) on the SAME full matrix and
block width, serial whole-matrix spmv on all host cores.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SELL-C-sigma SpMMV GFLOP/s and HBM GB/s vs roofline at 1/2/4/8 B200"
UNIT = "GFLOP/s"
# sources of the SpMMV kernels: a traffic figure is reported only for the build it was captured on
KERNEL_SOURCES = ["paper_1507_08101_b200/csrc/spmv_kernels.cuh", "paper_1507_08101_b200/csrc/tma.cuh",
                  "paper_1507_08101_b200/csrc/ops.cuh", "paper_1507_08101_b200/csrc/spmv.cu"]


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", "--edge", dest="n", type=int, default=400, help="grid edge of the 3-D 7-point stencil")
    p.add_argument("--width", type=int, default=8)
    p.add_argument("--chunk", type=int, default=32)
    p.add_argument("--sigma", type=int, default=256)
    p.add_argument("--halo", default="auto", choices=["auto", "ipc", "nccl"], help="halo transport at N > 1")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-planes", type=int, default=0,
                   help="z-planes of a bounded CPU sample (0 = the full matrix, same config)")
    p.add_argument("--cpu-reps", type=int, default=5)
    p.add_argument("--ref-max-steps", type=int, default=40, help="cap on the reference arm's timed steps")
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


def kernel_source_hash() -> str:
    h = hashlib.sha256()
    for rel in KERNEL_SOURCES:
        with open(os.path.join(ROOT, rel), "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def captured_traffic(key: str):
    """DRAM bytes per launch from the committed ncu capture of THIS kernel build
    (profiles/ncu_traffic.json entries carry the source hash they were taken on)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as f:
        tr = json.load(f)
    e = tr.get(key)
    if not isinstance(e, dict):
        return None, None
    src = kernel_source_hash()
    if e.get("source_hash") != src:
        return None, {"capture": e.get("capture"), "stale": True, "source_hash": src,
                      "captured_on": e.get("source_hash")}
    return float(e["dram_bytes"]), {"capture": e.get("capture"), "source_hash": src,
                                    "read": e.get("dram_read"), "write": e.get("dram_write")}


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

def cpu_reference(args, steps: int, warmup: int):
    """The reference's own CPU library (oracle/_ref, built from /root/reference by
    oracle/Makefile.ref) through its public C ABI: sellkit_crs_create ->
    sellkit_mat_build -> sellkit_spmv on the whole matrix, all host cores.  The
    matrix is the full n^3 stencil (the same config as the GPU line) unless
    --cpu-planes asks for a bounded box sample.  Falls back to the oracle port
    (single thread) only when the reference build is absent."""
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    os.environ.setdefault("SELLKIT_NUM_WORKERS", str(cores))
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    from oracle.oracle import REF_LIB_PATH, FullSize, Oracle, hash_block, stencil_box
    n, width = args.n, args.width
    t_setup = time.perf_counter()
    if args.cpu_planes and args.cpu_planes < n:
        rowptr, col, val = stencil_box(n, n, args.cpu_planes)
        sample = f"3-D 7-pt box {n}x{n}x{args.cpu_planes} ({len(rowptr) - 1} rows, {int(rowptr[-1])} nnz)"
    else:
        rowptr, col, val = FullSize().stencil7_crs(n)
        sample = f"full {n}^3 matrix ({len(rowptr) - 1} rows, {int(rowptr[-1])} nnz), same as the GPU config"
    nrows = len(rowptr) - 1
    nnz = int(rowptr[-1])
    sample += f", SELL-{args.chunk}-{args.sigma}, w={width}, y = A x, whole-matrix serial spmv"
    flops = 2.0 * nnz * width
    times = []
    if os.path.exists(REF_LIB_PATH):
        from paper_1507_08101_b200 import sellkit
        xv = FullSize().hash_block(nrows, width, 42)
        ref = sellkit.Sellkit(REF_LIB_PATH, ext=False)
        ref.call("sellkit_set_num_workers", int(os.environ["SELLKIT_NUM_WORKERS"]))
        crs = ref.crs(rowptr, col, val)
        del rowptr, col, val
        tb = time.perf_counter()
        A = crs.build(args.chunk, args.sigma)
        t_build = time.perf_counter() - tb
        tb = time.perf_counter()
        ref.call("sellkit_mat_update_values", A.h, crs.h)
        t_update = time.perf_counter() - tb
        del crs
        x = ref.densemat_from(xv)
        del xv
        y = ref.densemat(nrows, width)
        setup_s = time.perf_counter() - t_setup
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            ref.spmv(y, A, x)
            if i >= warmup:
                times.append(time.perf_counter() - t0)
        kind, used = "reference", int(os.environ["OMP_NUM_THREADS"])
    else:
        t_build = t_update = None
        xv = hash_block(nrows, width, 42)
        orc = Oracle()
        A = orc.build(rowptr, col, val, args.chunk, args.sigma)
        setup_s = time.perf_counter() - t_setup
        for i in range(1 + max(1, steps // 3)):
            t0 = time.perf_counter()
            orc.spmv(A, xv)
            if i >= 1:
                times.append(time.perf_counter() - t0)
        kind, used = "port", 1
    t = float(np.median(times))
    construction = None
    if t_build is not None:
        construction = {"build_ms": t_build * 1e3, "update_values_ms": t_update * 1e3,
                        "spmv_units_build": t_build / t, "spmv_units_update_values": t_update / t}
    return {"value": flops / t / 1e9, "unit": UNIT, "cores": used, "kind": kind, "sample": sample,
            "ms_per_step": t * 1e3, "steps": len(times), "setup_s": setup_s,
            "same_config": not (args.cpu_planes and args.cpu_planes < n), "construction": construction}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    steps = max(1, min(args.steps, args.ref_max_steps))
    cb = cpu_reference(args, steps, max(1, min(args.warmup, 3)))
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": cb["steps"], "warmup": max(1, min(args.warmup, 3)), "ms_per_step": cb["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"3-D 7-pt Laplacian {args.n}^3 ({args.n ** 3} rows, {stencil_nnz(args.n)} nnz), "
                               f"SELL-{args.chunk}-{args.sigma}, row-major block width {args.width}, y = A x",
                   "sample": cb["sample"], "same_config": cb["same_config"], "setup_s": cb["setup_s"],
                   "steps_requested": args.steps},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "construction": cb["construction"],
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_subprocess(args):
    """The reference arm in a fresh process (no CUDA context, no second OpenMP runtime
    beside torch's): the same number the driver's reference arm measures."""
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--gpus", "1", "--steps",
           str(args.cpu_reps), "--warmup", "1", "--n", str(args.n), "--width", str(args.width), "--chunk",
           str(args.chunk), "--sigma", str(args.sigma), "--cpu-planes", str(args.cpu_planes)]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE")}
    try:
        out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900).stdout
        line = json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])
        cb = dict(line["cpu_baseline"])
        cb["ms_per_step"] = line["ms_per_step"]
        cb["steps"] = line["steps"]
        cb["same_config"] = line["config"]["same_config"]
        cb["construction"] = line.get("construction")
        return cb
    except Exception as e:  # reported, never fatal for the GPU line
        return {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                "sample": f"unavailable: {type(e).__name__}: {e}"[:300]}


# -------------------------------------------------------------------- ours --

def run_ours(args, rank, world, local_rank):
    import torch
    from paper_1507_08101_b200 import sellkit

    ndev = torch.cuda.device_count()
    shared = world > ndev
    torch.cuda.set_device(local_rank % ndev)
    sk = sellkit.load()
    n, w = args.n, args.width
    N = n ** 3
    nnz_total = stencil_nnz(n)
    transport = None
    if world > 1 or os.environ.get("SELLKIT_BENCH_RANKCTX") == "1":
        # one process per GPU: rank context with the halo exchange; SELLKIT_BENCH_RANKCTX=1
        # exercises the same path at world size 1
        from paper_1507_08101_b200 import dist as skdist
        transport = None if args.halo == "auto" else args.halo
        job = skdist.bench_setup(sk, n, w, args.chunk, args.sigma, rank, world, transport=transport)
        transport = job.keep[0].transport
    else:
        job = None

    stream = torch.cuda.ExternalStream(sk.stream())
    build = None
    if job is None:
        crs = sk.crs_stencil(7, n)
        torch.cuda.synchronize()
        t_builds, t_updates = [], []
        for rep in range(3):  # the first build also pays the process's first big allocations
            t0 = time.perf_counter()
            A = crs.build(args.chunk, args.sigma)           # synchronous: SELL-C-sigma built on the GPU
            t_builds.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            sk.call("sellkit_mat_update_values", A.h, crs.h)  # constant-pattern value refresh
            t_updates.append(time.perf_counter() - t0)
            if rep < 2:
                del A
        build = {"build_ms": float(np.median(t_builds)) * 1e3, "update_values_ms": float(np.median(t_updates)) * 1e3,
                 "build_ms_each": [t * 1e3 for t in t_builds]}
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

    def barrier():
        if world > 1:
            import torch.distributed as tdist
            tdist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        import torch.distributed as tdist
        t = torch.tensor([v], dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    sk.set_sync(False)
    for _ in range(args.warmup):
        step()
    sk.synchronize()
    torch.cuda.synchronize()
    barrier()
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
    barrier()
    clk = clocks.stop() if rank == 0 else None
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    total_ms = max_over_ranks(evs[0].elapsed_time(evs[-1]))
    sk.set_sync(True)
    ms_per_step = total_ms / args.steps
    flops_step = 2.0 * nnz_total * w
    value = flops_step / (ms_per_step * 1e-3) / 1e9

    # algorithmic bytes: 12 B/nnz + x read + y write (+ received halo), per GPU
    halo_bytes = job.halo_bytes if job is not None else 0
    alg_bytes = 12.0 * nnz_local + 8.0 * w * rows_local * 2 + halo_bytes
    kernel_ms = float(np.mean(per_step)) if job is None else job.kernel_ms(per_step)
    peak, peak_kind = measured_peaks()
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
    traffic, traffic_src = captured_traffic(f"n{n}_w{w}_C{args.chunk}_s{args.sigma}_g{world}")

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
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        if job is not None and job.e2e_flush is not None:
            job.e2e_flush()
        e1.record(stream)
        torch.cuda.synchronize()
        sk.set_sync(True)
        te = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps)
        e2e = {"value": flops_step / (te * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(h2d) * world,
               "d2h_bytes_per_step": int(d2h) * world, "ms_per_step": te, "steps": args.e2e_steps,
               "path": ("sellkit_spmv on view_plain host buffers (pinned), streamed H2D/sweep/D2H"
                        if job is None else "per rank: H2D x, sellkit_ext_rank_spmv, D2H y; consecutive steps "
                        "overlap the upload with the previous download")}

    if job is not None:
        torch.cuda.synchronize()
        job.close()  # collective: no rank frees IPC slots / leaves NCCL while a peer still uses them
    if rank != 0:
        return
    cb = None
    if not args.no_cpu_baseline:
        cb = cpu_baseline_subprocess(args)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"3-D 7-pt Laplacian {n}^3 ({N} rows, {nnz_total} nnz), SELL-{args.chunk}-{args.sigma}, "
                               f"row-major block width {w}, y = A x",
                   "rows": N, "nnz": nnz_total, "block_width": w, "chunk_height": args.chunk, "sigma": args.sigma,
                   "parallelism": f"rows{world}", "halo_transport": transport,
                   "gpus_shared": shared,
                   "l2": "inputs (13.6 GB) >> 126 MB L2, no flush needed",
                   "hbm_gbs_aggregate": alg_bytes * world / (ms_per_step * 1e-3) / 1e9},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_kind": peak_kind,
                     "alg_bytes_per_launch": alg_bytes, "kernel_ms": kernel_ms},
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "cpu_baseline": cb,
    }
    if build is not None:
        # the paper's construction metric (perfmodel.cpp:41-45): cost in SpMV units
        build["spmv_units_build"] = build["build_ms"] / ms_per_step
        build["spmv_units_update_values"] = build["update_values_ms"] / ms_per_step
        build["what"] = ("median wall time of 3 synchronous sellkit_mat_build calls (CRS in HBM -> SELL-C-sigma: "
                         "sigma-sort, permutation, chunk lengths/offsets, fill) and sellkit_mat_update_values, over "
                         "ms_per_step; the 2nd and 3rd build reuse the freed matrix's device memory through the "
                         "library's buffer cache (build_ms_each[0]: with the driver allocations)")
        line["construction"] = build
    print(json.dumps(line), flush=True)


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` outside torchrun: start N ranks (one process per GPU)
    through torch.distributed.run on this node.  Needs N visible GPUs;
    SELLKIT_BENCH_SHARE_GPUS=1 lets ranks share GPUs (protocol checks only -- the
    line then says gpus_shared and is not a scaling measurement)."""
    import torch
    ndev = torch.cuda.device_count()
    if ndev < args.gpus and os.environ.get("SELLKIT_BENCH_SHARE_GPUS") != "1":
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {ndev}", file=sys.stderr)
        return 1
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    # torch.distributed.run's parser takes "--n" for an abbreviation of its own options: pass
    # the grid edge under its unambiguous name
    fwd = ["--edge" if a == "--n" else ("--edge=" + a[4:] if a.startswith("--n=") else a) for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + fwd
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world != args.gpus and rank == 0:
        print(f"bench.py: note: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)",
              file=sys.stderr)
    if world > 1:
        import torch.distributed as tdist
        # CPU plumbing only (setup handshake, barriers, max over ranks); the halo moves
        # through the library's own transport
        tdist.init_process_group("gloo")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as tdist
            tdist.destroy_process_group()


if __name__ == "__main__":
    main()
