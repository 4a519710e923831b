"""One rank of the multi-process distributed SpMMV tests (tests/test_dist_mp_gpu.py).

Launched once per rank (RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT in the
environment) with a gloo process group for the setup handshake only; the halo
and the dots move through the library's CUDA-IPC transport.  Every rank of a
test runs on the same (single) GPU: the ranks' streams wait on each other only
through stream memory operations, never inside a kernel.

For each golden case of tests/golden/dist.npz with k == WORLD_SIZE, this rank
builds its row block from the golden CRS (global columns), connects, and runs
the plain sweep (three dots) and the fused cases f1/f2 four times each (eager,
graph capture, graph replay, eager with SMs reserved for the halo pack), writing its rows of y / z (original order) and
the dots to <outdir>/rank<r>.npz for the parent test to compare.
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    outdir, cases = sys.argv[1], sys.argv[2].split(",")
    transport = sys.argv[3] if len(sys.argv) > 3 else "ipc"
    import torch
    import torch.distributed as tdist
    from paper_1507_08101_b200 import dist, sellkit

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank % torch.cuda.device_count())
    tdist.init_process_group("gloo")
    sk = sellkit.load()
    g = np.load(os.path.join(ROOT, "tests", "golden", "dist.npz"))
    out = {}
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from fused_cases import FUSED  # (name, flags, gamma) of the fused golden cases
    for key in cases:
        name = key.split("|")[0]
        C_, sigma = int(key.split("|")[3]), int(key.split("|")[4])
        rp, col, val = g[f"{name}|crs|rowptr"], g[f"{name}|crs|col"], g[f"{name}|crs|val"]
        n = len(rp) - 1
        off = g[key + "|row_offset"]
        r0, r1 = int(off[rank]), int(off[rank + 1])
        b, e = rp[r0], rp[r1]
        rows = sk.crs(rp[r0:r1 + 1] - b, col[b:e], val[b:e], ncols=n)
        rc = dist.setup_rank(sk, rows, off, rank, world, C_, sigma, transport=transport, max_width=2)
        assert rc.transport == transport, rc.transport
        perm = rc.row_perm()
        nl = r1 - r0
        w = 2

        def stored(a):
            s = np.empty((nl, w))
            s[perm] = a[r0:r1]
            return s
        yd, zd = sk.densemat(nl, w), sk.densemat(nl, w)
        dots_dev = torch.zeros(3 * w, dtype=torch.float64, device="cuda")
        runs = [("plain", sellkit.DOT_YY | sellkit.DOT_XY | sellkit.DOT_XX, None, g[key + "|x"], None, None)]
        for fname, flags, gam in FUSED:
            fk = f"{key}|{fname}"
            runs.append((fname, flags, gam, g[fk + "|x"], g[fk + "|y0"], g[fk + "|z0"]))
        for fname, flags, gam, xv, y0, z0 in runs:
            xd = sk.densemat_from(stored(xv))
            keep = []

            def sc(v):
                a = np.ascontiguousarray(np.atleast_1d(v), np.float64)
                keep.append(a)
                return sellkit._ptr(a)
            o = sellkit.spmv_opts()
            sk.lib.sellkit_spmv_opts_init(C.byref(o))
            o.flags = flags
            if fname != "plain":
                o.alpha, o.beta, o.delta, o.eta = sc(0.5), sc(-1.0), sc(1.0), sc(0.3)
                if flags & sellkit.VSHIFT:
                    gl = torch.tensor(gam, dtype=torch.float64, device="cuda")  # device list: graphable
                    keep.append(gl)
                    o.gamma = C.c_void_p(gl.data_ptr())
                else:
                    o.gamma = sc(gam[0])
            o.dot = C.c_void_p(dots_dev.data_ptr())
            for rep in range(4):  # eager, capture + replay, replay, eager with SMs left to the pack
                if rep == 3:
                    rc.set_options(graphs=0, reserve_sms=16)
                if y0 is not None:
                    yd.copy_in(stored(y0))
                    zd.copy_in(stored(z0))
                dots_dev.zero_()
                torch.cuda.synchronize()
                sk.call("sellkit_ext_rank_spmv", yd.h, rc.h, xd.h, C.byref(o),
                        zd.h if flags & sellkit.CHAIN_AXPBY else None, 0)
                torch.cuda.synchronize()
                ys, zs = yd.copy_out(), zd.copy_out()
                out[f"{key}|{fname}|{rep}|y"] = ys[perm]
                out[f"{key}|{fname}|{rep}|z"] = zs[perm]
                out[f"{key}|{fname}|{rep}|dot"] = dots_dev.cpu().numpy()
            rc.set_options(graphs=1, reserve_sms=0)
        out[f"{key}|stats"] = np.array([rc.stats()["bytes"], rc.stats()["msgs"]], np.int64)
        rc.close()  # collective: waits for every rank before freeing the exported slots
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    tdist.barrier()
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
