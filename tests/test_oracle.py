"""Pin the CPU oracle (oracle/sellkit_oracle.c + oracle/oracle.py) against the
reference: the reference's own known-answer tests and golden fixtures produced
by the reference build (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle.oracle import build_context, hash_block, random_crs, stencil_crs

LAYOUT_KEYS = ["row_perm_inv", "row_perm", "rowlen", "chunk_len", "chunk_offset", "val", "col"]


def golden_mats(g):
    names = sorted({k.split("|")[0] for k in g.files if "|crs|" in k})
    return {n: (g[f"{n}|crs|rowptr"], g[f"{n}|crs|col"], g[f"{n}|crs|val"], int(g[f"{n}|crs|ncols"][0]))
            for n in names}


# ------------------------------------------------------------ known answers

def test_sigma_permutation_kats(orc):
    # proj/tests/unit_sparse.cpp:75-89
    assert orc.sigma_permutation([1, 2, 1, 3], 4).tolist() == [3, 1, 0, 2]
    assert orc.sigma_permutation([1, 2, 1, 3], 1).tolist() == [0, 1, 2, 3]
    assert orc.sigma_permutation([2, 2, 2, 2, 2], 5).tolist() == [0, 1, 2, 3, 4]
    assert orc.sigma_permutation([1, 3, 1, 5], 2).tolist() == [1, 0, 3, 2]


def test_worked_4x4_layout(orc):
    # proj/tests/unit_sparse.cpp:91-113
    A = orc.build([0, 1, 3, 4, 7], [0, 0, 1, 2, 1, 2, 3], np.arange(1, 8, dtype=float), 2, 4)
    L = A.layout()
    assert L["chunk_len"].tolist() == [3, 1]
    assert L["chunk_offset"].tolist() == [0, 6, 8]
    assert L["val"][:6].tolist() == [5, 2, 6, 3, 7, 0]
    assert L["val"][6:8].tolist() == [1, 4]
    assert L["beta"] == pytest.approx(0.875)
    assert L["row_perm_inv"].tolist() == [3, 1, 0, 2]
    assert L["col"][5] == 0


def test_build_validation(orc):
    # proj/tests/unit_sparse.cpp:144-154
    rp, c, v = [0, 1, 3, 4, 7], [0, 0, 1, 2, 1, 2, 3], np.arange(1, 8, dtype=float)
    with pytest.raises(ValueError):
        orc.build(rp, c, v, 0, 1)
    with pytest.raises(ValueError):
        orc.build(rp, c, v, 4, 2)
    orc.build(rp, c, v, 4, 4)
    orc.build(rp, c, v, 3, 7)
    with pytest.raises(ValueError):
        orc.build(rp, [9] + c[1:], v, 2, 1)


def test_partition_kats(orc):
    # proj/tests/unit_runtime.cpp:470-492 style: equal weights, rounding, clamps
    assert orc.partition(10, 2).tolist() == [0, 5, 10]
    assert orc.partition(10, 2, weights=[1, 2.3333333]).tolist() == [0, 3, 10]
    assert orc.partition(4, 4).tolist() == [0, 1, 2, 3, 4]


# ------------------------------------------------------- golden fixtures

def test_layouts_match_reference(orc, golden):
    g = golden("sell_layouts.npz")
    mats = golden_mats(g)
    combos = sorted({tuple(k.split("|")[:3]) for k in g.files if "|crs|" not in k})
    assert len(combos) > 50
    for name, C, sigma in combos:
        rp, c, v, nc = mats[name]
        L = orc.build(rp, c, v, int(C), int(sigma), ncols=nc).layout()
        for key in LAYOUT_KEYS:
            ref = g[f"{name}|{C}|{sigma}|{key}"]
            assert np.array_equal(L[key], ref), (name, C, sigma, key)
        assert L["beta"] == g[f"{name}|{C}|{sigma}|beta"][0]


def test_fused_spmv_matches_reference_bitwise(orc, golden):
    g = golden("spmv.npz")
    gl = golden("sell_layouts.npz")
    rp, c, v, nc = golden_mats(gl)["rand0"]
    A = orc.build(rp, c, v, 4, 8)
    x, y0, z0 = g["fusion|x"], g["fusion|y0"], g["fusion|z0"]
    gammas = np.array([0.5, -1.5, 2.0])
    n_checked = 0
    for flags in range(128):
        if (flags & 0x02) and (flags & 0x04):
            continue
        y, z, dots = orc.spmv(A, x, y0, z0, flags, alpha=1.3, beta=-0.7, gamma=0.5, gamma_list=gammas, delta=0.4,
                              eta=2.2, workers=1)
        assert np.array_equal(y, g[f"fusion|{flags}|y"]), flags
        assert np.array_equal(z, g[f"fusion|{flags}|z"]), flags
        ref_dots = g[f"fusion|{flags}|dot"]
        for s, bit in enumerate((0x08, 0x10, 0x20)):
            if flags & bit:
                assert np.array_equal(dots[s * 3:(s + 1) * 3], ref_dots[s * 3:(s + 1) * 3]), flags
        n_checked += 1
    assert n_checked == 96


def test_sweeps_match_reference_bitwise(orc, golden):
    g = golden("spmv.npz")
    mats = golden_mats(golden("sell_layouts.npz"))
    keys = sorted({tuple(k.split("|")[1:5]) for k in g.files if k.startswith("sweep|")})
    assert keys
    for name, C, sigma, w in keys:
        rp, c, v, nc = mats[name]
        A = orc.build(rp, c, v, int(C), int(sigma), ncols=nc)
        key = f"sweep|{name}|{C}|{sigma}|{w}"
        y, _, dots = orc.spmv(A, g[key + "|x"], flags=0x38, workers=1)
        assert np.array_equal(y, g[key + "|y"]), key
        assert np.array_equal(dots, g[key + "|dot"]), key


def test_tsm_matches_reference_bitwise(orc, golden):
    g = golden("tsm.npz")
    shapes = sorted({tuple(k.split("|")[:3]) for k in g.files})
    for n, m, k in shapes:
        key = f"{n}|{m}|{k}"
        V, W, X = g[key + "|V"], g[key + "|W"], g[key + "|X"]
        for a, b in [(1.0, 0.0), (0.5, -1.25)]:
            assert np.array_equal(orc.tsmttsm(V, W, X, a, b, workers=1), g[key + f"|tsmttsm|{a}|{b}"]), key
            assert np.array_equal(orc.tsmm(V, X, W, a, b), g[key + f"|tsmm|{a}|{b}"]), key


def test_kahan_cancellation(orc):
    # proj/tests/unit_sparse.cpp:625-636: [1e16, 1, -1e16] -> 1 with Kahan, 0 without
    v = np.ones((3, 1))
    w = np.array([[1e16], [1.0], [-1e16]])
    assert orc.tsmttsm(v, w, kahan=True)[0, 0] == 1.0
    assert orc.tsmttsm(v, w, kahan=False)[0, 0] == 0.0


def test_dist_metadata_matches_reference(orc, golden):
    g = golden("dist.npz")
    names = sorted({k.split("|")[0] for k in g.files if "|crs|" in k})
    cases = sorted({tuple(k.split("|")[:5]) for k in g.files if "|crs|" not in k})
    assert cases
    for name, k, by_nnz, C, sigma in cases:
        assert name in names
        rp, c, v = g[f"{name}|crs|rowptr"], g[f"{name}|crs|col"], g[f"{name}|crs|val"]
        row_offset, ranks = build_context(rp, c, v, int(k), int(C), int(sigma), orc, by_nnz=bool(int(by_nnz)))
        key = f"{name}|{k}|{by_nnz}|{C}|{sigma}"
        assert np.array_equal(row_offset, g[key + "|row_offset"]), key
        for r, sm in enumerate(ranks):
            p = f"{key}|r{r}."
            assert np.array_equal(sm["halo_cols"], g[p + "halo_cols"]), (key, r)
            assert np.array_equal(sm["halo_owner"], g[p + "halo_owner"]), (key, r)
            assert np.array_equal(sm["recv_owner"], g[p + "recv_owner"]), (key, r)
            assert np.array_equal(sm["recv_count"], g[p + "recv_count"]), (key, r)
            assert sm["send_to"] == g[p + "send_to"].tolist(), (key, r)
            rows = np.concatenate(sm["send_rows"]) if sm["send_rows"] else np.zeros(0, np.int32)
            assert np.array_equal(rows, g[p + "send_rows"]), (key, r)
            L = sm["local"].layout()
            for kk in LAYOUT_KEYS:
                assert np.array_equal(L[kk], g[p + "local." + kk]), (key, r, kk)
            assert (sm["remote"] is not None) == bool(g[p + "has_remote"][0])
            if sm["remote"] is not None:
                R = sm["remote"].layout()
                for kk in LAYOUT_KEYS:
                    assert np.array_equal(R[kk], g[p + "remote." + kk]), (key, r, kk)


def test_generators():
    rp, c, v = stencil_crs(7, 4)
    assert rp[-1] == 7 * 4 ** 3 - 6 * 4 ** 2
    rp, c, v = stencil_crs(5, 10)
    assert rp[-1] == 5 * 100 - 4 * 10
    rng = np.random.default_rng(0)
    rp, c, v = random_crs(rng, 30, 30, 0.1)
    assert np.all(np.diff(rp) >= 1)
    h = hash_block(4, 3, 42)
    assert h.shape == (4, 3) and np.all(np.abs(h) < 1)
