"""Host-side logic of the row distribution, no GPU: partition, the per-rank split
(halo columns, owners, receive counts) and the send lists, produced by the C
library's host-only planner (sellkit_ext_rankplan_*) and, for the multi-process
protocol, exchanged over torch.distributed (gloo, world size 2) -- all checked
against the oracle's restatement of partition.hpp, which test_oracle.py pins to
the reference."""
import os
import socket

import numpy as np
import pytest

from oracle.oracle import build_context, random_crs, stencil_crs
from paper_1507_08101_b200 import dist, sellkit


def test_partition_kats(sk, orc):
    # proj/tests/unit_runtime.cpp:470-492 style cases through the C ABI, vs the oracle
    for n, k, w, by_nnz in [(10, 2, None, False), (10, 2, [1, 2.3333333], False), (4, 4, None, False),
                            (100, 7, None, False), (1000, 8, [1, 2, 3, 4, 5, 6, 7, 8], False)]:
        assert dist.partition(sk, n, k, w).tolist() == orc.partition(n, k, w).tolist()
    lens = np.random.default_rng(1).integers(1, 9, 500)
    assert dist.partition(sk, 500, 5, by_nnz=True, rowlens=lens).tolist() == \
        orc.partition(500, 5, by_nnz=True, rowlens=lens).tolist()
    with pytest.raises(sellkit.SellkitError):
        dist.partition(sk, 3, 4)  # more ranks than rows


def _plans_for(sk, rowptr, col, val, off):
    plans = []
    for r in range(len(off) - 1):
        r0, r1 = off[r], off[r + 1]
        b, e = rowptr[r0], rowptr[r1]
        plans.append(dist.RankPlan(sk, rowptr[r0:r1 + 1] - b, col[b:e], val[b:e], off, r))
    return plans


@pytest.mark.parametrize("case", ["stencil", "random", "tri"])
@pytest.mark.parametrize("k", [2, 3, 4, 7])
def test_rank_plans_match_oracle(sk, orc, case, k):
    rng = np.random.default_rng(k)
    if case == "stencil":
        rowptr, col, val = stencil_crs(7, 7)
    elif case == "random":
        rowptr, col, val = random_crs(rng, 90, 90, 0.05)
    else:
        n = 10
        rows = [[c for c in (r - 1, r, r + 1) if 0 <= c < n] for r in range(n)]
        rowptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
        col = np.concatenate(rows).astype(np.int64)
        val = np.ones(len(col))
    off, ranks = build_context(rowptr, col, val, k, 4, 8, orc)
    plans = _plans_for(sk, rowptr, col, val, off)
    # single-process send-list assembly (partition.hpp:268-277)
    for r, p in enumerate(plans):
        for owner, cols in p.requests().items():
            plans[owner].set_sends(r, cols)
    for r, (p, sm) in enumerate(zip(plans, ranks)):
        req = p.requests()
        assert sorted(req) == sm["recv_owner"].tolist()
        if len(sm["halo_cols"]):
            assert np.array_equal(np.concatenate([req[o] for o in sorted(req)]), sm["halo_cols"])
        for o, cnt in zip(sm["recv_owner"], sm["recv_count"]):
            assert len(req[o]) == cnt
        sends = p.sends()
        assert sorted(sends) == sm["send_to"]
        # oracle send lists are stored rows; the plan holds local rows (before the sigma order)
        perm_inv = sm["local"].layout()["row_perm_inv"]
        for to, rows in zip(sm["send_to"], sm["send_rows"]):
            assert np.array_equal(perm_inv[rows], sends[to])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, q):
    import torch.distributed as tdist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        tdist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.oracle import Oracle
        orc = Oracle()
        sk = sellkit.load()
        rowptr, col, val = stencil_crs(7, 6)
        off, ranks = build_context(rowptr, col, val, world, 8, 32, orc)
        r0, r1 = off[rank], off[rank + 1]
        b, e = rowptr[r0], rowptr[r1]
        plan = dist.RankPlan(sk, rowptr[r0:r1 + 1] - b, col[b:e], val[b:e], off, rank)
        incoming = dist.exchange_requests(plan.requests(), rank, world)
        for to in sorted(incoming):
            plan.set_sends(to, incoming[to])
        sm = ranks[rank]
        sends = plan.sends()
        perm_inv = sm["local"].layout()["row_perm_inv"]
        ok = sorted(sends) == sm["send_to"] and all(
            np.array_equal(perm_inv[rows], sends[to]) for to, rows in zip(sm["send_to"], sm["send_rows"]))
        tdist.destroy_process_group()
        q.put((rank, ok, ""))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(exc)))


def test_multiprocess_request_exchange_gloo():
    """The one-process-per-GPU setup protocol over torch.distributed (gloo, world size 2)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, msg in res:
        assert ok, (rank, msg)


def _gather_worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as tdist
        tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        from paper_1507_08101_b200.dist import gather_in_rank_order
        t = torch.full((3, 2), float(rank + 1), dtype=torch.float64)
        parts = gather_in_rank_order(t)
        ok = len(parts) == world and all(bool(torch.all(p == r + 1)) for r, p in enumerate(parts))
        tdist.destroy_process_group()
        q.put((rank, ok, ""))
    except Exception as exc:  # pragma: no cover
        q.put((rank, False, repr(exc)))


def test_tsmttsm_partials_gathered_in_rank_order_gloo():
    """Sharded TSMTTSM plumbing: every rank receives all m x k partials
    in rank order (gloo, world size 3), so the ordered sum is identical on every rank."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, msg in res:
        assert ok, (rank, msg)
