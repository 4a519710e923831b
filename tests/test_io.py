"""Matrix-file ingestion (Matrix Market, GCRS binary) against the reference.

Fixtures (tests/golden/io.npz, made by tests/golden/make_io_golden.py) hold the
reference's GCRS bytes for each Matrix Market case, or its error code; the
GPU tests require our reader + writer to produce the same bytes (bit-exact CRS:
row pointers, columns, values) and the same error codes.  Mirrors the
reference's io tests (proj/tests/unit_basic.cpp:336-479)."""
import os

import numpy as np
import pytest

from oracle.oracle import REF_LIB_PATH

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
IO_ERR = 5


def _cases(g):
    for i, name in enumerate(g["names"]):
        text = bytes(g["text"][g["text_off"][i]:g["text_off"][i + 1]])
        gcrs = bytes(g["gcrs"][g["gcrs_off"][i]:g["gcrs_off"][i + 1]])
        yield str(name), int(g["dts"][i]), text, int(g["errs"][i]), gcrs


@pytest.mark.skipif(not os.path.exists(REF_LIB_PATH), reason="oracle/_ref not built")
def test_fixtures_pinned_to_reference(golden, tmp_path):
    """The committed fixtures are what the reference library produces (CPU)."""
    from oracle.oracle import RefIO
    ref = RefIO()
    g = golden("io.npz")
    mm, gb = str(tmp_path / "a.mtx"), str(tmp_path / "a.gcrs")
    for name, dt, text, err, gcrs in _cases(g):
        with open(mm, "wb") as f:
            f.write(text)
        r = ref.mm_to_gcrs(mm, dt, gb)
        if err:
            assert r == err, name
        else:
            assert r == gcrs, name


@pytest.mark.gpu
def test_matrix_market_bit_exact(sk, golden, tmp_path):
    from paper_1507_08101_b200.sellkit import SellkitError
    g = golden("io.npz")
    mm, gb = str(tmp_path / "a.mtx"), str(tmp_path / "a.gcrs")
    for name, dt, text, err, gcrs in _cases(g):
        with open(mm, "wb") as f:
            f.write(text)
        if err:
            with pytest.raises(SellkitError) as ei:
                sk.crs_read_mm(mm, dt)
            assert ei.value.code == err, name
            continue
        A = sk.crs_read_mm(mm, dt)
        A.write_bin(gb)
        with open(gb, "rb") as f:
            assert f.read() == gcrs, name


@pytest.mark.gpu
def test_reference_unit_cases(sk, tmp_path):
    """proj/tests/unit_basic.cpp:336-372: value-level checks through the device CRS."""
    mm = str(tmp_path / "a.mtx")
    with open(mm, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n2 1 5.0\n")
    A = sk.crs_read_mm(mm)
    assert A.dims() == (2, 2, 2)
    # a SELL-1-1 build is the CRS itself (unit_sparse.cpp:122-133)
    L = A.build(1, 1).export()
    assert list(L["col"]) == [1, 0] and list(L["val"]) == [5.0, 5.0]


@pytest.mark.gpu
def test_binary_round_trip_and_rejects(sk, golden, tmp_path):
    from paper_1507_08101_b200.sellkit import SellkitError
    g = golden("io.npz")
    narrow, wide = bytes(g["bin_narrow"]), bytes(g["bin_wide"])
    src, out = str(tmp_path / "in.gcrs"), str(tmp_path / "out.gcrs")
    for data in (narrow, wide):
        with open(src, "wb") as f:
            f.write(data)
        A = sk.crs_read_bin(src)
        assert A.dt == 1 and A.dims()[:2] == (17, 13)
        A.write_bin(out)
        assert open(out, "rb").read() == narrow
        A.write_bin(out, wide_cols=True)
        assert open(out, "rb").read() == wide

    def rejects(data, code=IO_ERR):
        with open(src, "wb") as f:
            f.write(data)
        with pytest.raises(SellkitError) as ei:
            sk.crs_read_bin(src)
        assert ei.value.code == code

    rejects(b"XXXX" + narrow[4:])                     # wrong magic
    rejects(narrow[:-8])                              # truncated payload
    rejects(narrow + b"zz")                           # trailing bytes
    rejects(narrow[:4] + b"\x02\x00\x00\x00" + narrow[8:])  # unknown version
    rejects(b"")                                      # empty
    # header nnz inconsistent with the row pointers
    bad = bytearray(narrow)
    bad[32] ^= 1
    rejects(bytes(bad))
    # columns out of order inside a row pass the I/O checks but fail validation
    nrows = 17
    col0 = 4 + 4 + 4 + 24 + (nrows + 1) * 8
    rp = np.frombuffer(narrow[36:36 + (nrows + 1) * 8], np.int64)
    r = int(np.argmax(np.diff(rp) >= 2))
    k = int(rp[r])
    cols = bytearray(narrow)
    a, b = cols[col0 + 4 * k:col0 + 4 * k + 4], cols[col0 + 4 * k + 4:col0 + 4 * k + 8]
    cols[col0 + 4 * k:col0 + 4 * k + 4], cols[col0 + 4 * k + 4:col0 + 4 * k + 8] = b, a
    rejects(bytes(cols), code=1)
    with pytest.raises(SellkitError) as ei:
        sk.crs_read_bin(str(tmp_path / "missing.gcrs"))
    assert ei.value.code == IO_ERR


@pytest.mark.gpu
def test_mm_to_spmv_matches_oracle(sk, orc, tmp_path):
    """A Matrix Market matrix goes through build + spmv like any CRS."""
    rng = np.random.default_rng(3)
    n = 300
    rows = rng.integers(1, n + 1, 2000)
    cols = rng.integers(1, n + 1, 2000)
    vals = rng.standard_normal(2000)
    mm = str(tmp_path / "r.mtx")
    with open(mm, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n" + f"{n} {n} {len(vals)}\n")
        for r, c, v in zip(rows, cols, vals):
            f.write(f"{r} {c} {v:.17g}\n")
    A = sk.crs_read_mm(mm)
    gb = str(tmp_path / "r.gcrs")
    A.write_bin(gb)
    raw = open(gb, "rb").read()
    nnz = int(np.frombuffer(raw[28:36], np.uint64)[0])
    rp = np.frombuffer(raw[36:36 + (n + 1) * 8], np.int64)
    col = np.frombuffer(raw[36 + (n + 1) * 8:36 + (n + 1) * 8 + 4 * nnz], np.uint32).astype(np.int64)
    val = np.frombuffer(raw[36 + (n + 1) * 8 + 4 * nnz:], np.float64)
    M = A.build(32, 64)
    x = np.random.default_rng(4).standard_normal((n, 8))
    X, Y = sk.densemat_from(x), sk.densemat(n, 8)
    sk.spmv(Y, M, X)
    yo, _, _ = orc.spmv(orc.build(rp, col, val, 32, 64), x)
    assert np.array_equal(Y.copy_out(), yo)
