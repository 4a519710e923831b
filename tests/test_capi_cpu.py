"""C-ABI boundary checks that need no GPU: the B200 library loads, exports every
symbol include/*.h declares, and its host-only entry points behave like the
reference's (proj/tests/unit_capi.cpp)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1507_08101_b200 import sellkit

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"\btypedef\b[^;]*;", "", text, flags=re.S)  # function-pointer types are not functions
    names = set(re.findall(r"\b(sellkit_\w+)\s*\(", text))
    # typedef'd function pointer names are not functions
    return sorted(n for n in names if n not in {"sellkit_row_fn", "sellkit_task_fn"})


def exported_symbols(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_library_exports_every_declared_symbol(sk):
    syms = exported_symbols(sk.path)
    for header in ("sellkit.h", "sellkit_ext.h"):
        decl = declared_functions(header)
        assert decl, header
        missing = [d for d in decl if d not in syms]
        assert not missing, (header, missing)
    # and nothing but the API is exported (hidden visibility)
    assert all(s.startswith("sellkit_") for s in syms), sorted(s for s in syms if not s.startswith("sellkit_"))


def test_binding_covers_headers(sk):
    decl = set(declared_functions("sellkit.h")) | set(declared_functions("sellkit_ext.h"))
    bound = set(sellkit.API_NAMES) | set(sellkit.EXT_NAMES)
    assert decl == bound, (decl ^ bound)


def test_header_compiles_as_c99(tmp_path):
    # proj/tests/c_api_compile.c: the header is plain C
    src = tmp_path / "t.c"
    src.write_text('#include "sellkit.h"\n#include "sellkit_ext.h"\nint main(void){sellkit_spmv_opts o; '
                   'sellkit_spmv_opts_init(&o); return (int)o.flags;}\n')
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-c", "-I", os.path.join(ROOT, "include"), str(src),
                    "-o", str(tmp_path / "t.o")], check=True)


def test_error_names_and_narrow_index(sk):
    # unit_capi.cpp:26-32
    assert sk.lib.sellkit_error_name(0) == b"ok"
    out = C.c_int32(-1)
    assert sk.lib.sellkit_narrow_index(5, C.byref(out)) == 0 and out.value == 5
    assert sk.lib.sellkit_narrow_index(1 << 31, C.byref(out)) == sellkit.ERR_OVERFLOW
    assert sk.lib.sellkit_narrow_index(-1, C.byref(out)) == sellkit.ERR_INVALID_ARG


def test_select_kernel_cascade(sk):
    # unit_capi.cpp:333-342 and unit_sparse.cpp:468-486
    assert sk.select_kernel(32, 4) == (32, 4, 1)
    c, w, _ = sk.select_kernel(7, 1000)
    assert (c, w) == (0, 0)
    assert sk.select_kernel(7, 4)[0] == 0
    assert sk.select_kernel(32, 1000)[:2] == (32, 0)
    assert sk.select_kernel(32, 4, sellkit.COL_MAJOR) == (0, 0, 0)
    assert sk.select_kernel(32, 64) == (32, 64, 1)


def test_buildconfig(sk):
    p, n = C.POINTER(C.c_int)(), C.c_size_t()
    sk.call("sellkit_buildconfig_chunk_heights", C.byref(p), C.byref(n))
    assert [p[i] for i in range(n.value)] == [4, 8, 32]
    sk.call("sellkit_buildconfig_block_widths", C.byref(p), C.byref(n))
    assert [p[i] for i in range(n.value)] == [1, 2, 4, 8, 16, 32, 64]


def test_perf_model(sk):
    # unit_capi.cpp:296-322
    v = C.c_double()
    sk.call("sellkit_spmv_code_balance", sellkit.R64, 4, 0, 0.0, C.byref(v))
    assert v.value == 6.0
    sk.call("sellkit_index_width_saving", 4, C.byref(v))
    assert v.value == pytest.approx(1.0 / 3.0)
    assert sk.lib.sellkit_index_width_saving(7, C.byref(v)) == sellkit.ERR_UNSUPPORTED
    sk.call("sellkit_roofline_bound", 50.0, 176.0, 6.0, C.byref(v))
    assert v.value == pytest.approx(50.0 / 6.0)
    sk.call("sellkit_crs_refresh_cost", 100, 8, 1200.0, C.byref(v))
    assert v.value == pytest.approx(2.0)
    sk.call("sellkit_spmv_code_balance", sellkit.C64, 4, 0, 0.0, C.byref(v))
    assert v.value == 2.5
    sk.call("sellkit_spmv_code_balance", sellkit.R32, 4, 0, 0.0, C.byref(v))
    assert v.value == 4.0


def test_region_table_golden(sk):
    r = C.c_void_p()
    sk.call("sellkit_region_create", b"spmv (GF/s)", C.byref(r))
    for _ in range(100):
        sk.call("sellkit_region_record", r, 16.4)
    t = C.c_void_p()
    arr = (C.c_void_p * 1)(r)
    sk.call("sellkit_region_table", arr, 1, C.byref(t))
    text = C.cast(t, C.c_char_p).value.decode()
    sk.lib.sellkit_string_free(t)
    assert "Region      | Calls |    P_max | P_skip10" in text
    assert "spmv (GF/s) |   100 | 1.64e+01 | 1.64e+01" in text
    # reference golden: proj/tests/golden/spmvbench_identity.txt line format
    r2 = C.c_void_p()
    sk.call("sellkit_region_create", b"spmv (GF/s)", C.byref(r2))
    for _ in range(100):
        sk.call("sellkit_region_record", r2, 2.0e-3)
    arr = (C.c_void_p * 1)(r2)
    sk.call("sellkit_region_table", arr, 1, C.byref(t))
    text = C.cast(t, C.c_char_p).value.decode()
    sk.lib.sellkit_string_free(t)
    assert "spmv (GF/s) |   100 | 2.00e-03 | 2.00e-03" in text
    p = C.c_double()
    assert sk.lib.sellkit_region_p_skip10(r2, C.byref(p)) == 0 and p.value == pytest.approx(2e-3)
    sk.lib.sellkit_region_destroy(r)
    sk.lib.sellkit_region_destroy(r2)


def test_task_pool_is_unsupported(sk):
    out = C.c_void_p()
    assert sk.lib.sellkit_pool_create(2, None, 0, C.byref(out)) == sellkit.ERR_UNSUPPORTED
    assert out.value is None


def test_num_workers_and_timer(sk):
    sk.call("sellkit_set_num_workers", 3)
    assert sk.lib.sellkit_num_workers() == 3
    assert sk.lib.sellkit_set_num_workers(0) == sellkit.ERR_INVALID_ARG
    t0 = sk.lib.sellkit_now_seconds()
    assert t0 > 0


def test_pencil_order_is_a_block_permutation():
    """orders.pencil_order: a permutation of the row blocks; consecutive z of one y-slab
    are adjacent in the sweep (the property that shrinks the RHS reuse window)."""
    import numpy as np
    from paper_1507_08101_b200.orders import pencil_order
    lx, ly, lz, per = 64, 8, 6, 4
    o = pencil_order(lx, ly, lz, per_site=per, block_rows=256, yb=2)
    nblocks = lx * ly * lz * per // 256
    assert sorted(o.tolist()) == list(range(nblocks))
    bpl = lx * per // 256
    # first slab: y in {0, 1}, all z, before any y >= 2
    first = o[: lz * 2 * bpl]
    ys = (first // bpl) % ly
    assert set(ys.tolist()) == {0, 1}
    import pytest
    with pytest.raises(ValueError):
        pencil_order(10, 4, 4, per_site=1, block_rows=32)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                    "oracle", "_ref", "libsellkit.so")),
                    reason="oracle/_ref not built")
def test_perf_model_equals_reference_library(sk):
    """Host-side perf model (perfmodel.cpp:11-45) against the reference library itself
    (oracle/_ref) over a grid of inputs: identical doubles and error codes."""
    from oracle.oracle import REF_LIB_PATH
    ref = C.CDLL(REF_LIB_PATH)
    ref.sellkit_spmv_code_balance.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_double)]
    ref.sellkit_roofline_bound.argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]
    ref.sellkit_crs_refresh_cost.argtypes = [C.c_int64, C.c_int, C.c_double, C.POINTER(C.c_double)]
    ref.sellkit_index_width_saving.argtypes = [C.c_int, C.POINTER(C.c_double)]
    a, b = C.c_double(), C.c_double()
    for dt in (sellkit.R32, sellkit.R64, sellkit.C32, sellkit.C64):
        for ib in (2, 4, 8, 3):
            for vec in (0, 1):
                for nnzr in (0.0, 1.0, 7.0, 13.5):
                    e1 = sk.lib.sellkit_spmv_code_balance(dt, ib, vec, nnzr, C.byref(a))
                    e2 = ref.sellkit_spmv_code_balance(dt, ib, vec, nnzr, C.byref(b))
                    assert e1 == e2 and (e1 != 0 or a.value == b.value), (dt, ib, vec, nnzr)
    for bw, pk, cb in [(50.0, 176.0, 6.0), (6465.8, 37000.0, 1.895), (1.0, 1.0, 0.0), (-1.0, 2.0, 3.0)]:
        e1 = sk.lib.sellkit_roofline_bound(bw, pk, cb, C.byref(a))
        e2 = ref.sellkit_roofline_bound(bw, pk, cb, C.byref(b))
        assert e1 == e2 and (e1 != 0 or a.value == b.value)
    for nnz, vb, bw in [(100, 8, 1200.0), (447040000, 8, 6465.8), (0, 16, 1.0), (5, 3, 2.0)]:
        e1 = sk.lib.sellkit_crs_refresh_cost(nnz, vb, bw, C.byref(a))
        e2 = ref.sellkit_crs_refresh_cost(nnz, vb, bw, C.byref(b))
        assert e1 == e2 and (e1 != 0 or a.value == b.value)
    for vb in (1, 2, 4, 8, 16, 7):
        e1 = sk.lib.sellkit_index_width_saving(vb, C.byref(a))
        e2 = ref.sellkit_index_width_saving(vb, C.byref(b))
        assert e1 == e2 and (e1 != 0 or a.value == b.value)
