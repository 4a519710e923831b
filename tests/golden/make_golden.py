"""Generate golden fixtures from the REFERENCE implementation itself.

Runs in the build container only (needs /root/reference and oracle/_ref built by
`make -f oracle/Makefile.ref`).  Writes small .npz files next to this script;
they are committed and are the parity anchor for tests/ on machines without
the reference (the GPU box).

    python tests/golden/make_golden.py

Sources of truth:
  * oracle/_ref/refdump (our exporter compiled against the reference's own
    sellcs.hpp / partition.hpp) for SELL layouts and distribution metadata;
  * oracle/_ref/libsellkit.so through its public C ABI (driven by the same
    ctypes binding as the B200 library) for spmv / tsm / dist results.
Inputs are seeded numpy draws, stored in the fixtures.
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import REF_LIB_PATH, REFDUMP_PATH, random_crs, stencil_crs  # noqa: E402
from paper_1507_08101_b200 import sellkit as sk  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def write_crs(path, rowptr, col, val, ncols):
    with open(path, "wb") as f:
        np.array([len(rowptr) - 1, ncols, rowptr[-1]], np.int64).tofile(f)
        np.asarray(rowptr, np.int64).tofile(f)
        np.asarray(col, np.int64).tofile(f)
        np.asarray(val, np.float64).tofile(f)


def read_records(path):
    out = {}
    dt = {0: np.int32, 1: np.int64, 2: np.float64}
    with open(path, "rb") as f:
        data = f.read()
    pos = 0
    while pos < len(data):
        nl = int(np.frombuffer(data, np.int32, 1, pos)[0]); pos += 4
        name = data[pos:pos + nl].decode(); pos += nl
        code = int(np.frombuffer(data, np.int32, 1, pos)[0]); pos += 4
        cnt = int(np.frombuffer(data, np.int64, 1, pos)[0]); pos += 8
        t = dt[code]
        out[name] = np.frombuffer(data, t, cnt, pos).copy(); pos += cnt * np.dtype(t).itemsize
    return out


def refdump(*args):
    with tempfile.TemporaryDirectory() as td:
        crs_path = os.path.join(td, "a.bin")
        out_path = os.path.join(td, "out.bin")
        rowptr, col, val, ncols = args[0]
        write_crs(crs_path, rowptr, col, val, ncols)
        cmd = [REFDUMP_PATH, args[1], crs_path] + [str(a) for a in args[2:]] + [out_path]
        subprocess.run(cmd, check=True)
        return read_records(out_path)


def example_4x4():
    # proj/tests/unit_sparse.cpp:19-27
    return (np.array([0, 1, 3, 4, 7]), np.array([0, 0, 1, 2, 1, 2, 3]), np.arange(1, 8, dtype=float), 4)


def matrices():
    rng = np.random.default_rng(20240601)
    mats = {"ex4": example_4x4()}
    for i, (n, d) in enumerate([(37, 0.15), (150, 0.08), (203, 0.05)]):
        rp, c, v = random_crs(rng, n, n, d)
        mats[f"rand{i}"] = (rp, c, v, n)
    rp, c, v = stencil_crs(5, 12)
    mats["lap2d_12"] = (rp, c, v, 144)
    rp, c, v = stencil_crs(7, 6)
    mats["lap3d_6"] = (rp, c, v, 216)
    # irregular row lengths (heavy permutation): lengths 1..40
    lens = rng.integers(1, 41, 120)
    rows = [np.sort(rng.choice(120, size=l, replace=False)) for l in lens]
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    mats["ragged"] = (rp, np.concatenate(rows).astype(np.int64), rng.uniform(-1, 1, rp[-1]), 120)
    return mats


def gen_layouts(mats):
    out = {}
    params = [(1, 1), (2, 1), (2, 4), (4, 1), (4, 4), (4, 8), (8, 32), (32, 1), (32, 64), (32, 256), (3, 7)]
    for name, m in mats.items():
        n = len(m[0]) - 1
        for C, sigma in params + [(8, n), (32, n)]:
            if not (sigma == 1 or sigma % C == 0 or sigma >= n):
                continue
            rec = refdump(m, "sell", C, sigma)
            for k, v in rec.items():
                out[f"{name}|{C}|{sigma}|{k}"] = v
    for name, m in mats.items():
        out[f"{name}|crs|rowptr"] = np.asarray(m[0], np.int64)
        out[f"{name}|crs|col"] = np.asarray(m[1], np.int64)
        out[f"{name}|crs|val"] = np.asarray(m[2], np.float64)
        out[f"{name}|crs|ncols"] = np.array([m[3]], np.int64)
    np.savez_compressed(os.path.join(OUT, "sell_layouts.npz"), **out)
    print("sell_layouts.npz:", len(out), "arrays")


def ref_lib():
    return sk.Sellkit(REF_LIB_PATH, ext=False, strict=True)


def storage_vec(perm, logical):
    """logical rows -> storage rows: out[perm[i]] = logical[i]."""
    out = np.empty_like(logical)
    out[perm] = logical
    return out


def gen_spmv(mats):
    ref = ref_lib()
    ref.call("sellkit_set_num_workers", 1)
    rng = np.random.default_rng(7)
    out = {}
    # fusion equivalence over all 96 flag combinations (unit_sparse.cpp:364-439)
    rp, c, v, n = mats["rand0"]
    A = ref.crs(rp, c, v, n).build(4, 8)
    w = 3
    xv, yv, zv = (rng.uniform(-1, 1, (n, w)) for _ in range(3))
    out["fusion|x"], out["fusion|y0"], out["fusion|z0"] = xv, yv, zv
    alpha, beta, delta, eta = 1.3, -0.7, 0.4, 2.2
    gammas = np.array([0.5, -1.5, 2.0])
    for flags in range(128):
        if (flags & sk.SHIFT) and (flags & sk.VSHIFT):
            continue
        x = ref.densemat_from(xv)
        y = ref.densemat_from(yv)
        z = ref.densemat_from(zv)
        dots = np.full(3 * w, 99.0)
        gam = gammas if flags & sk.VSHIFT else gammas[:1]
        ref.spmv(y, A, x, flags=flags, alpha=alpha, beta=beta, gamma=gam, delta=delta, eta=eta, z=z, dot=dots)
        out[f"fusion|{flags}|y"] = y.copy_out()
        out[f"fusion|{flags}|z"] = z.copy_out()
        out[f"fusion|{flags}|dot"] = dots
    # widths / chunk heights on the stencils and a ragged matrix (storage space)
    for name, C, sigma in [("lap3d_6", 32, 256), ("lap2d_12", 32, 1), ("ragged", 8, 32), ("rand1", 4, 16),
                           ("rand2", 32, 203), ("lap3d_6", 3, 12)]:
        rp, c, v, n = mats[name]
        A = ref.crs(rp, c, v, n).build(C, sigma)
        for w in (1, 2, 3, 4, 8, 16):
            xv = rng.uniform(-1, 1, (n, w))
            x = ref.densemat_from(xv)
            y = ref.densemat(n, w)
            dots = np.zeros(3 * w)
            ref.spmv(y, A, x, flags=sk.DOT_YY | sk.DOT_XY | sk.DOT_XX, dot=dots)
            key = f"sweep|{name}|{C}|{sigma}|{w}"
            out[key + "|x"], out[key + "|y"], out[key + "|dot"] = xv, y.copy_out(), dots
    np.savez_compressed(os.path.join(OUT, "spmv.npz"), **out)
    print("spmv.npz:", len(out), "arrays")


def gen_tsm():
    ref = ref_lib()
    ref.call("sellkit_set_num_workers", 1)
    rng = np.random.default_rng(11)
    out = {}
    for n, m, k in [(100, 1, 1), (257, 2, 3), (300, 4, 4), (129, 8, 8), (64, 3, 5), (500, 16, 16)]:
        V, W, X = rng.uniform(-1, 1, (n, m)), rng.uniform(-1, 1, (n, k)), rng.uniform(-1, 1, (m, k))
        key = f"{n}|{m}|{k}"
        out[key + "|V"], out[key + "|W"], out[key + "|X"] = V, W, X
        for a, b in [(1.0, 0.0), (0.5, -1.25)]:
            xo, vd, wd, xd = (ref.densemat_from(X), ref.densemat_from(V), ref.densemat_from(W),
                              ref.densemat_from(X))
            av, bv = np.array([a]), np.array([b])
            ref.call("sellkit_tsmttsm", xo.h, vd.h, wd.h, av.ctypes.data, bv.ctypes.data, 0)
            out[key + f"|tsmttsm|{a}|{b}"] = xo.copy_out()
            wo = ref.densemat_from(W)
            ref.call("sellkit_tsmm", wo.h, vd.h, xd.h, av.ctypes.data, bv.ctypes.data)
            out[key + f"|tsmm|{a}|{b}"] = wo.copy_out()
    np.savez_compressed(os.path.join(OUT, "tsm.npz"), **out)
    print("tsm.npz:", len(out), "arrays")


from fused_cases import FUSED as FUSED_DIST  # noqa: E402  (name, flags, gamma)


def gen_dist(mats):
    out = {}
    ref = ref_lib()
    ref.call("sellkit_set_num_workers", 1)
    rng = np.random.default_rng(5)
    # tridiagonal n=10 (unit_capi.cpp:153-226)
    n = 10
    rows = [[c for c in (r - 1, r, r + 1) if 0 <= c < n] for r in range(n)]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])])
    col = np.concatenate(rows)
    val = np.array([2.0 if c == r else -1.0 for r, rr in enumerate(rows) for c in rr])
    cases = {"tri10": (rp, col, val, n), "rand1": mats["rand1"], "lap3d_6": mats["lap3d_6"], "ragged": mats["ragged"]}
    for name, m in cases.items():
        for k, by_nnz, C, sigma in [(1, 0, 2, 2), (2, 0, 2, 2), (3, 0, 4, 8), (4, 1, 8, 32), (7, 0, 4, 4)]:
            if k > len(m[0]) - 1:
                continue
            rec = refdump(m, "dist", k, by_nnz, C, sigma)
            key = f"{name}|{k}|{by_nnz}|{C}|{sigma}"
            for kk, vv in rec.items():
                out[f"{key}|{kk}"] = vv
            # dist_spmv results through the reference C ABI (NO_OVERLAP), w = 2
            crs = ref.crs(m[0], m[1], m[2], m[3])
            ctx = sk.vp()
            wts = np.ones(k)
            ref.call("sellkit_ctx_create", crs.h, wts.ctypes.data, k, by_nnz, C, sigma, 1, sk.C.byref(ctx))
            w = 2
            xv = rng.uniform(-1, 1, (len(m[0]) - 1, w))
            xg = ref.densemat_from(xv)
            yg = ref.densemat(len(m[0]) - 1, w)
            dx, dy = sk.vp(), sk.vp()
            ref.call("sellkit_dvec_create", ctx, w, 0, sk.C.byref(dx))
            ref.call("sellkit_dvec_create", ctx, w, 0, sk.C.byref(dy))
            ref.call("sellkit_dvec_scatter", ctx, xg.h, dx)
            o = sk.spmv_opts()
            dots = np.zeros(3 * w)
            o.flags = sk.DOT_YY | sk.DOT_XY | sk.DOT_XX
            o.dot = dots.ctypes.data
            ref.call("sellkit_dist_spmv", dy, ctx, dx, sk.C.byref(o), 0, None, 1)
            ref.call("sellkit_dvec_gather", ctx, dy, yg.h)
            bytes_, msgs = sk.C.c_uint64(), sk.C.c_uint64()
            ref.call("sellkit_ctx_comm_stats", ctx, sk.C.byref(bytes_), sk.C.byref(msgs))
            out[f"{key}|x"], out[f"{key}|y"], out[f"{key}|dot"] = xv, yg.copy_out(), dots
            out[f"{key}|comm"] = np.array([bytes_.value, msgs.value], np.int64)
            # fused flags through dist_spmv (own RNG stream: the arrays above stay as they were)
            for fname, flags, gam in FUSED_DIST:
                frng = np.random.default_rng(1000 + 31 * k + sum(map(ord, name)) + (0 if fname == "f1" else 7))
                x2, y0, z0 = (frng.uniform(-1, 1, (len(m[0]) - 1, w)) for _ in range(3))
                dz = sk.vp()
                ref.call("sellkit_dvec_create", ctx, w, 0, sk.C.byref(dz))
                gx2, gy0, gz0 = ref.densemat_from(x2), ref.densemat_from(y0), ref.densemat_from(z0)
                ref.call("sellkit_dvec_scatter", ctx, gx2.h, dx)
                ref.call("sellkit_dvec_scatter", ctx, gy0.h, dy)
                ref.call("sellkit_dvec_scatter", ctx, gz0.h, dz)
                sc = {nm: np.array(vv, np.float64) for nm, vv in
                      [("alpha", [0.5]), ("beta", [-1.0]), ("delta", [1.0]), ("eta", [0.3]), ("gamma", gam)]}
                fo = sk.spmv_opts()
                fo.flags = flags
                fo.alpha, fo.beta, fo.delta, fo.eta, fo.gamma = (sc[nm].ctypes.data for nm in
                                                                 ("alpha", "beta", "delta", "eta", "gamma"))
                fdots = np.zeros(3 * w)
                fo.dot = fdots.ctypes.data
                ref.call("sellkit_dist_spmv", dy, ctx, dx, sk.C.byref(fo), 0, dz, 1)
                zg = ref.densemat(len(m[0]) - 1, w)
                ref.call("sellkit_dvec_gather", ctx, dy, yg.h)
                ref.call("sellkit_dvec_gather", ctx, dz, zg.h)
                fk = f"{key}|{fname}"
                out[fk + "|x"], out[fk + "|y0"], out[fk + "|z0"] = x2, y0, z0
                out[fk + "|y"], out[fk + "|z"], out[fk + "|dot"] = yg.copy_out(), zg.copy_out(), fdots
                ref.lib.sellkit_dvec_destroy(dz)
            ref.lib.sellkit_dvec_destroy(dx)
            ref.lib.sellkit_dvec_destroy(dy)
            ref.lib.sellkit_ctx_destroy(ctx)
        for kk in ("rowptr", "col", "val"):
            pass
        out[f"{name}|crs|rowptr"] = np.asarray(m[0], np.int64)
        out[f"{name}|crs|col"] = np.asarray(m[1], np.int64)
        out[f"{name}|crs|val"] = np.asarray(m[2], np.float64)
    np.savez_compressed(os.path.join(OUT, "dist.npz"), **out)
    print("dist.npz:", len(out), "arrays")


if __name__ == "__main__":
    mats = matrices()
    gen_layouts(mats)
    gen_spmv(mats)
    gen_tsm()
    gen_dist(mats)
