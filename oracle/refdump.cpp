// refdump -- golden-fixture exporter built against the REFERENCE's internal
// headers (/root/reference/proj/src, see oracle/Makefile.ref).  Test
// infrastructure only.  The reference's C ABI has no getter for the SELL-C-sigma
// arrays or the split-matrix/halo metadata, so this tool builds them with the
// reference's own templates and writes them out for tests/golden/make_golden.py:
//
//   refdump sell  <crs.bin> <C> <sigma> <out.bin>
//       sellkit::build (sellcs.hpp:236-246) -> row_perm_inv, row_perm, rowlen,
//       chunk_len, chunk_offset, val, col, beta
//   refdump dist  <crs.bin> <nranks> <by_nnz> <C> <sigma> <out.bin>
//       DistContext::build_context (partition.hpp:250-286) -> row_offset and,
//       per rank, halo columns/owners, recv counts, send lists and both parts
//
// crs.bin: int64 nrows, ncols, nnz; int64 rowptr[nrows+1]; int64 col[nnz];
//          double val[nnz].
// out.bin: repeated records {int32 name_len; char name[]; int32 dtype
//          (0=i32,1=i64,2=f64); int64 count; payload}.

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "partition.hpp"
#include "sellcs.hpp"

using namespace sellkit;

namespace {

CrsData<double> read_crs(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) { std::perror(path); std::exit(2); }
    int64_t hdr[3];
    if (std::fread(hdr, sizeof(int64_t), 3, f) != 3) std::exit(2);
    CrsData<double> a;
    a.nrows = hdr[0];
    a.ncols = hdr[1];
    a.rowptr.resize(std::size_t(hdr[0]) + 1);
    a.col.resize(std::size_t(hdr[2]));
    a.val.resize(std::size_t(hdr[2]));
    bool ok = std::fread(a.rowptr.data(), 8, a.rowptr.size(), f) == a.rowptr.size();
    ok = ok && std::fread(a.col.data(), 8, a.col.size(), f) == a.col.size();
    ok = ok && std::fread(a.val.data(), 8, a.val.size(), f) == a.val.size();
    std::fclose(f);
    if (!ok) { std::fprintf(stderr, "short read %s\n", path); std::exit(2); }
    return a;
}

struct Writer {
    FILE* f;
    explicit Writer(const char* path) : f(std::fopen(path, "wb")) {
        if (!f) { std::perror(path); std::exit(2); }
    }
    ~Writer() { std::fclose(f); }
    void put(const std::string& name, int dtype, const void* data, int64_t count, int esize) {
        int32_t nl = int32_t(name.size());
        std::fwrite(&nl, 4, 1, f);
        std::fwrite(name.data(), 1, name.size(), f);
        std::fwrite(&dtype, 4, 1, f);
        std::fwrite(&count, 8, 1, f);
        if (count) std::fwrite(data, std::size_t(esize), std::size_t(count), f);
    }
    template <class V>
    void i32(const std::string& n, const V& v) { put(n, 0, v.data(), int64_t(v.size()), 4); }
    template <class V>
    void i64(const std::string& n, const V& v) { put(n, 1, v.data(), int64_t(v.size()), 8); }
    template <class V>
    void f64(const std::string& n, const V& v) { put(n, 2, v.data(), int64_t(v.size()), 8); }
};

void dump_sell(Writer& w, const std::string& p, const SellMatrix<double>& m) {
    w.i32(p + "row_perm_inv", m.row_perm_inv);
    w.i32(p + "row_perm", m.row_perm);
    w.i32(p + "rowlen", m.rowlen);
    w.i32(p + "chunk_len", m.chunk_len);
    w.i64(p + "chunk_offset", m.chunk_offset);
    w.f64(p + "val", m.val);
    w.i32(p + "col", m.col);
    std::vector<double> beta{m.beta};
    w.f64(p + "beta", beta);
    std::vector<int32_t> dims{m.nrows, m.ncols, m.nrows_padded, m.cols_permuted ? 1 : 0};
    w.i32(p + "dims", dims);
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: refdump sell|dist ...\n");
        return 2;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "sell" && argc == 6) {
            auto a = read_crs(argv[2]);
            SellParams p{std::atoi(argv[3]), std::atoi(argv[4])};
            auto m = build(a, p);
            Writer w(argv[5]);
            dump_sell(w, "", m);
            return 0;
        }
        if (cmd == "dist" && argc == 8) {
            auto a = read_crs(argv[2]);
            const int k = std::atoi(argv[3]);
            RankWeights rw;
            rw.weights.assign(std::size_t(k), 1.0);
            rw.mode = std::atoi(argv[4]) ? WeightMode::by_nnz : WeightMode::by_rows;
            SellParams p{std::atoi(argv[5]), std::atoi(argv[6])};
            auto ctx = DistContext<double>::build_context(a, rw, p, false);
            Writer w(argv[7]);
            w.i64("row_offset", ctx.plan.row_offset);
            for (int r = 0; r < k; ++r) {
                const auto& sm = ctx.ranks[r];
                const std::string pre = "r" + std::to_string(r) + ".";
                std::vector<int64_t> hcols, howners, rc_owner, rc_count;
                for (auto& [o, c] : sm.halo_map) { howners.push_back(o); hcols.push_back(c); }
                for (auto& [o, n] : sm.recv_counts) { rc_owner.push_back(o); rc_count.push_back(n); }
                w.i64(pre + "halo_cols", hcols);
                w.i64(pre + "halo_owner", howners);
                w.i64(pre + "recv_owner", rc_owner);
                w.i64(pre + "recv_count", rc_count);
                std::vector<int64_t> sl_to, sl_len;
                std::vector<int32_t> sl_rows;
                for (auto& sl : sm.send_lists) {
                    sl_to.push_back(sl.to);
                    sl_len.push_back(int64_t(sl.rows.size()));
                    sl_rows.insert(sl_rows.end(), sl.rows.begin(), sl.rows.end());
                }
                w.i64(pre + "send_to", sl_to);
                w.i64(pre + "send_len", sl_len);
                w.i32(pre + "send_rows", sl_rows);
                dump_sell(w, pre + "local.", sm.local);
                std::vector<int32_t> hr{sm.has_remote ? 1 : 0};
                w.i32(pre + "has_remote", hr);
                if (sm.has_remote) dump_sell(w, pre + "remote.", sm.remote);
            }
            return 0;
        }
    } catch (const Error& e) {
        std::fprintf(stderr, "refdump: sellkit error %d: %s\n", int(e.code()), e.what());
        return 3;
    }
    std::fprintf(stderr, "refdump: bad arguments\n");
    return 2;
}
