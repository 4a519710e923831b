"""Golden fixtures for the matrix-file I/O path, produced by the REFERENCE.

Each case is a Matrix Market text (the reference tests' cases from
proj/tests/unit_basic.cpp:336-421 plus wider coverage: every field x symmetry,
array files, duplicates, comments, blank lines, exponent / signed / many-digit
values, float and complex element types) read by the reference's
`sellkit_crs_read_mm` (oracle/_ref/libsellkit.so) and written back by its
`sellkit_crs_write_bin`.  The fixture stores the MM text, the element type and
the reference's GCRS bytes (or its error code).  A seeded random matrix is also
written as narrow and wide GCRS by the reference for the binary reader.

Runs in the build container only (needs oracle/_ref):

    python tests/golden/make_io_golden.py
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import RefIO, random_crs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
R32, R64, C32, C64 = 0, 1, 2, 3


def cases():
    c = []
    add = lambda name, dt, text: c.append((name, dt, text))  # noqa: E731
    # proj/tests/unit_basic.cpp:336-421
    add("coord_basic", R64, "%%MatrixMarket matrix coordinate real general\n% comment line\n2 2 2\n1 1 1.0\n2 2 2.0\n")
    add("sym_expand", R64, "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n2 1 5.0\n")
    add("pattern_dups", R64, "%%MatrixMarket matrix coordinate pattern general\n2 3 3\n1 1\n1 1\n2 3\n")
    add("hermitian", C64, "%%MatrixMarket matrix coordinate complex hermitian\n2 2 2\n1 1 2.0 0.0\n2 1 1.0 3.0\n")
    add("skew", R64, "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 4.0\n")
    add("array", R64, "%%MatrixMarket matrix array real general\n2 2\n1.0\n3.0\n2.0\n4.0\n")
    add("bad_banner", R64, "not a matrix market file\n")
    add("bad_range", R64, "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    # wider coverage
    add("case_insensitive", R64, "%%MatrixMarket MATRIX Coordinate REAL General\n3 3 3\n3 3 -1e-3\n1 2 +2.5E2\n2 1 .5\n")
    add("blank_and_comments", R64,
        "%%MatrixMarket matrix coordinate real general\n%\n\n  % indented comment\n3 4 4\n\n1 4 1\n"
        "% mid comment\n3 1 0.1\n2 2 -0.0\n3 4 123456789.123456789\n")
    add("integer_field", R64, "%%MatrixMarket matrix coordinate integer general\n2 2 3\n1 1 7\n2 1 -3\n1 2 0\n")
    add("dups_sum_order", R64,
        "%%MatrixMarket matrix coordinate real general\n1 2 4\n1 2 1e16\n1 1 3\n1 2 1\n1 2 -1e16\n")
    add("symmetric_diag", R64, "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 1\n3 1 2\n2 2 3\n3 2 4\n")
    add("skew_diag_error", R64, "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n1 1 4.0\n")
    add("complex_general", C64,
        "%%MatrixMarket matrix coordinate complex general\n2 3 3\n1 3 1.5 -2.5\n2 1 0 1\n1 1 -1 0\n")
    add("complex_into_real", R64, "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 1\n")
    add("real_into_complex", C64, "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 2\n2 1 -1\n")
    add("pattern_symmetric", R64, "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 3\n")
    add("hermitian_real_field", C64, "%%MatrixMarket matrix coordinate real hermitian\n2 2 2\n1 1 1\n2 1 2\n")
    add("float_round", R32, "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 0.1\n2 2 3.14159265358979\n")
    add("cfloat", C32, "%%MatrixMarket matrix coordinate complex general\n1 2 2\n1 2 0.1 0.2\n1 1 -1 1e-40\n")
    add("array_symmetric", R64, "%%MatrixMarket matrix array real symmetric\n3 3\n1\n2\n3\n4\n5\n6\n")
    add("array_skew", R64, "%%MatrixMarket matrix array real skew-symmetric\n3 3\n1\n2\n3\n")
    add("array_complex", C64, "%%MatrixMarket matrix array complex general\n2 1\n1 2\n3 4\n")
    add("array_zeros_kept", R64, "%%MatrixMarket matrix array real general\n2 2\n0\n0\n1\n0\n")
    add("empty_rows", R64, "%%MatrixMarket matrix coordinate real general\n5 5 2\n5 1 1\n1 5 2\n")
    add("zero_nnz", R64, "%%MatrixMarket matrix coordinate real general\n3 2 0\n")
    add("truncated_entries", R64, "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 2\n")
    add("malformed_entry", R64, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1\n")
    add("missing_value", R64, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n")
    add("bad_field", R64, "%%MatrixMarket matrix coordinate quaternion general\n1 1 1\n1 1 1\n")
    add("array_pattern", R64, "%%MatrixMarket matrix array pattern general\n1 1\n1\n")
    add("missing_size", R64, "%%MatrixMarket matrix coordinate real general\n% only comments\n")
    add("empty_file", R64, "")
    add("zero_index", R64, "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1\n")
    rng = np.random.default_rng(11)
    lines = []
    n, m = 40, 33
    for _ in range(300):
        lines.append(f"{rng.integers(1, n + 1)} {rng.integers(1, m + 1)} {rng.standard_normal():.17g}")
    add("random_dups", R64, "%%MatrixMarket matrix coordinate real general\n" + f"{n} {m} {len(lines)}\n" +
        "\n".join(lines) + "\n")
    return c


def main():
    ref = RefIO()
    names, dts, texts, outs, errs = [], [], [], [], []
    with tempfile.TemporaryDirectory() as td:
        mm, gb = os.path.join(td, "a.mtx"), os.path.join(td, "a.gcrs")
        for name, dt, text in cases():
            with open(mm, "w") as f:
                f.write(text)
            r = ref.mm_to_gcrs(mm, dt, gb)
            names.append(name)
            dts.append(dt)
            texts.append(np.frombuffer(text.encode(), np.uint8))
            if isinstance(r, int):
                outs.append(np.zeros(0, np.uint8))
                errs.append(r)
            else:
                outs.append(np.frombuffer(r, np.uint8))
                errs.append(0)
        # binary reader input: a seeded random matrix through the reference writer
        rng = np.random.default_rng(5)
        rowptr, col, val = random_crs(rng, 17, 13, 0.2)
        lines = [f"{r + 1} {c + 1} {v:.17g}" for r in range(17) for c, v in
                 zip(col[rowptr[r]:rowptr[r + 1]], val[rowptr[r]:rowptr[r + 1]])]
        with open(mm, "w") as f:
            f.write("%%MatrixMarket matrix coordinate real general\n" + f"17 13 {len(lines)}\n" + "\n".join(lines) + "\n")
        narrow = ref.mm_to_gcrs(mm, R64, gb, wide=False)
        wide = ref.mm_to_gcrs(mm, R64, gb, wide=True)
        assert isinstance(narrow, bytes) and isinstance(wide, bytes), (narrow, wide)
    offs = np.cumsum([0] + [len(t) for t in texts])
    ooffs = np.cumsum([0] + [len(o) for o in outs])
    np.savez_compressed(
        os.path.join(OUT, "io.npz"),
        names=np.array(names), dts=np.array(dts, np.int32), errs=np.array(errs, np.int32),
        text=np.concatenate(texts), text_off=offs, gcrs=np.concatenate(outs), gcrs_off=ooffs,
        bin_narrow=np.frombuffer(narrow, np.uint8), bin_wide=np.frombuffer(wide, np.uint8))
    print("wrote io.npz:", len(names), "cases,", sum(e != 0 for e in errs), "error cases")


if __name__ == "__main__":
    main()
