// Matrix file input/output for the CRS handle (reference: proj/src/io.cpp,
// io.hpp; C ABI sellkit_crs_read_mm / _read_bin / _write_bin, capi.cpp).
//
// Host-side ingestion: the file is read in one piece, parsed on the host into
// CRS arrays with the reference's semantics, and handed to crs_from_host, which
// uploads and validates on the device (the CRS handle lives in HBM).
//
//  * Matrix Market (io.cpp:120-301): coordinate or array; real / integer /
//    complex / pattern; general / symmetric / skew-symmetric / hermitian.
//    Entries are 1-based; symmetric kinds are mirrored (skew negates, hermitian
//    conjugates, skew diagonals are an error); array files are column-major and
//    store the lower triangle for the symmetric kinds.  Entries are stably sorted
//    by (row, column) and duplicates summed in file order in double precision,
//    then converted to the element type (io.cpp:169-204).
//  * GCRS binary (io.hpp:12-28, io.cpp:303-356): "GCRS", u32 version 1, u32 flags
//    (bit0 complex, bit1 single, bit2 64-bit columns), u64 nrows, ncols, nnz,
//    u64 rowptr[nrows+1], u32|u64 col[nnz], values; little-endian, no trailing
//    bytes.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "objects.cuh"

namespace skb {

namespace {

// ------------------------------------------------------------ file helpers --

std::string slurp(const char* path) {
    SK_REQUIRE(path != nullptr, errc::invalid_arg, "null path");
    FILE* f = std::fopen(path, "rb");
    SK_REQUIRE(f != nullptr, errc::io, std::string("cannot open ") + path);
    std::string s;
    char buf[1 << 16];
    std::size_t n;
    while ((n = std::fread(buf, 1, sizeof(buf), f)) > 0) s.append(buf, n);
    const bool err = std::ferror(f) != 0;
    std::fclose(f);
    SK_REQUIRE(!err, errc::io, std::string("read failure on ") + path);
    return s;
}

// Line cursor over an in-memory file.
struct Lines {
    const std::string& s;
    std::size_t pos = 0;
    explicit Lines(const std::string& text) : s(text) {}
    bool next(const char*& b, const char*& e) {
        if (pos >= s.size()) return false;
        const std::size_t nl = s.find('\n', pos);
        const std::size_t end = nl == std::string::npos ? s.size() : nl;
        b = s.data() + pos;
        e = s.data() + end;
        pos = nl == std::string::npos ? s.size() : nl + 1;
        return true;
    }
    // next line that is neither blank nor a '%' comment (io.cpp:160-168)
    bool content(const char*& b, const char*& e) {
        while (next(b, e)) {
            const char* p = b;
            while (p < e && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
            if (p == e || *p == '%') continue;
            return true;
        }
        return false;
    }
};

// Whitespace-separated token reader on one line (formatted-extraction semantics:
// a field that does not parse fails the line).
struct Fields {
    const char* p;
    const char* e;
    Fields(const char* b, const char* end) : p(b), e(end) {}
    void skip() {
        while (p < e && std::isspace(static_cast<unsigned char>(*p))) ++p;
    }
    bool token(std::string& out) {
        skip();
        if (p == e) return false;
        const char* q = p;
        while (q < e && !std::isspace(static_cast<unsigned char>(*q))) ++q;
        out.assign(p, q);
        p = q;
        return true;
    }
    bool integer(gidx& v) {
        skip();
        if (p == e) return false;
        char tmp[32];
        const char* q = p;
        while (q < e && !std::isspace(static_cast<unsigned char>(*q))) ++q;
        const std::size_t n = std::min<std::size_t>(std::size_t(q - p), sizeof(tmp) - 1);
        std::memcpy(tmp, p, n);
        tmp[n] = 0;
        char* end = nullptr;
        errno = 0;
        const long long x = std::strtoll(tmp, &end, 10);
        if (end == tmp || errno == ERANGE) return false;
        p += end - tmp;
        v = gidx(x);
        return true;
    }
    bool real(double& v) {
        skip();
        if (p == e) return false;
        // decimal floating-point only, as formatted extraction accepts (no inf/nan/hex)
        const char c0 = *p;
        const char c1 = p + 1 < e ? p[1] : 0;
        const bool digit0 = std::isdigit(static_cast<unsigned char>(c0)) || c0 == '.';
        const bool signed_digit = (c0 == '+' || c0 == '-') &&
                                  (std::isdigit(static_cast<unsigned char>(c1)) || c1 == '.');
        if (!digit0 && !signed_digit) return false;
        char tmp[128];
        const char* q = p;
        while (q < e && !std::isspace(static_cast<unsigned char>(*q))) ++q;
        const std::size_t n = std::min<std::size_t>(std::size_t(q - p), sizeof(tmp) - 1);
        std::memcpy(tmp, p, n);
        tmp[n] = 0;
        char* end = nullptr;
        const double x = std::strtod(tmp, &end);
        if (end == tmp) return false;
        p += end - tmp;
        v = x;
        return true;
    }
};

std::string lower(std::string s) {
    for (auto& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

enum class MmField { real, integer, complex_, pattern };
enum class MmSym { general, symmetric, skew, hermitian };

struct MmBanner {
    bool coordinate = true;
    MmField field = MmField::real;
    MmSym sym = MmSym::general;
};

MmBanner parse_banner(const char* b, const char* e) {
    Fields f(b, e);
    std::string banner, object, format, field, sym;
    f.token(banner);
    f.token(object);
    f.token(format);
    f.token(field);
    f.token(sym);
    SK_REQUIRE(banner == "%%MatrixMarket", errc::io, "missing %%MatrixMarket banner");
    SK_REQUIRE(lower(object) == "matrix", errc::io, "only matrix objects are supported");
    MmBanner h;
    const std::string fm = lower(format);
    if (fm == "coordinate") h.coordinate = true;
    else if (fm == "array") h.coordinate = false;
    else fail(errc::io, "unknown Matrix Market format: " + format);
    const std::string fl = lower(field);
    if (fl == "real") h.field = MmField::real;
    else if (fl == "integer") h.field = MmField::integer;
    else if (fl == "complex") h.field = MmField::complex_;
    else if (fl == "pattern") h.field = MmField::pattern;
    else fail(errc::io, "unknown Matrix Market field: " + field);
    const std::string sy = lower(sym);
    if (sy == "general") h.sym = MmSym::general;
    else if (sy == "symmetric") h.sym = MmSym::symmetric;
    else if (sy == "skew-symmetric") h.sym = MmSym::skew;
    else if (sy == "hermitian") h.sym = MmSym::hermitian;
    else fail(errc::io, "unknown Matrix Market symmetry: " + sym);
    SK_REQUIRE(h.coordinate || h.field != MmField::pattern, errc::io, "array format cannot be pattern");
    return h;
}

// Coordinate triplets, kept as separate arrays; `seq` is the file order used as
// the stable-sort tie break.
struct Triplets {
    std::vector<gidx> row, col;
    std::vector<double> re, im;
    void push(gidx r, gidx c, double a, double b) {
        row.push_back(r);
        col.push_back(c);
        re.push_back(a);
        im.push_back(b);
    }
    std::size_t size() const { return row.size(); }
};

void store_value(unsigned char* dst, Datatype dt, double re, double im) {
    switch (dt) {
        case Datatype::r32: {
            const float v = static_cast<float>(re);
            std::memcpy(dst, &v, 4);
            break;
        }
        case Datatype::r64: std::memcpy(dst, &re, 8); break;
        case Datatype::c32: {
            const float v[2] = {static_cast<float>(re), static_cast<float>(im)};
            std::memcpy(dst, v, 8);
            break;
        }
        case Datatype::c64: {
            const double v[2] = {re, im};
            std::memcpy(dst, v, 16);
            break;
        }
    }
}

// io.cpp:169-204: range check, stable (row, col) order, duplicates summed.
std::unique_ptr<Crs> assemble(gidx nrows, gidx ncols, Triplets& t, Datatype dt) {
    const std::size_t n = t.size();
    for (std::size_t k = 0; k < n; ++k)
        SK_REQUIRE(t.row[k] >= 0 && t.row[k] < nrows && t.col[k] >= 0 && t.col[k] < ncols, errc::io,
                   "matrix market index out of range");
    std::vector<std::size_t> order(n);
    std::iota(order.begin(), order.end(), std::size_t(0));
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
        return t.row[a] != t.row[b] ? t.row[a] < t.row[b] : t.col[a] < t.col[b];
    });
    std::vector<gidx> rowptr(std::size_t(nrows) + 1, 0), col;
    std::vector<unsigned char> val;
    const std::size_t vb = value_bytes(dt);
    col.reserve(n);
    val.reserve(n * vb);
    std::size_t i = 0;
    while (i < n) {
        const gidx r = t.row[order[i]], c = t.col[order[i]];
        double re = 0.0, im = 0.0;
        while (i < n && t.row[order[i]] == r && t.col[order[i]] == c) {
            re += t.re[order[i]];
            im += t.im[order[i]];
            ++i;
        }
        if (!is_complex(dt)) SK_REQUIRE(im == 0.0, errc::io, "complex data cannot be read into a real matrix");
        col.push_back(c);
        const std::size_t at = val.size();
        val.resize(at + vb);
        store_value(val.data() + at, dt, re, im);
        rowptr[std::size_t(r) + 1]++;
    }
    for (gidx r = 0; r < nrows; ++r) rowptr[std::size_t(r) + 1] += rowptr[std::size_t(r)];
    return crs_from_host(dt, nrows, ncols, rowptr.data(), col.data(), val.data());
}

// ------------------------------------------------------------------ GCRS --

constexpr char kMagic[4] = {'G', 'C', 'R', 'S'};
constexpr std::uint32_t kVersion = 1;

struct Reader {
    const std::string& s;
    std::size_t pos = 0;
    explicit Reader(const std::string& b) : s(b) {}
    void need(std::size_t n) const {
        SK_REQUIRE(pos + n <= s.size(), errc::io, "truncated binary CRS file");
    }
    std::uint32_t u32() {
        need(4);
        std::uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= std::uint32_t(static_cast<unsigned char>(s[pos + i])) << (8 * i);
        pos += 4;
        return v;
    }
    std::uint64_t u64() {
        need(8);
        std::uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= std::uint64_t(static_cast<unsigned char>(s[pos + i])) << (8 * i);
        pos += 8;
        return v;
    }
};

void put32(std::string& o, std::uint32_t v) {
    for (int i = 0; i < 4; ++i) o.push_back(char((v >> (8 * i)) & 0xff));
}
void put64(std::string& o, std::uint64_t v) {
    for (int i = 0; i < 8; ++i) o.push_back(char((v >> (8 * i)) & 0xff));
}

}  // namespace

std::unique_ptr<Crs> crs_read_mm(const char* path, Datatype dt) {
    const std::string text = slurp(path);
    Lines lines(text);
    const char *b, *e;
    SK_REQUIRE(lines.next(b, e), errc::io, "empty file");
    const MmBanner h = parse_banner(b, e);
    SK_REQUIRE(lines.content(b, e), errc::io, "missing size line");
    SK_REQUIRE(h.field != MmField::complex_ || is_complex(dt), errc::io,
               "complex data cannot be read into a real matrix");
    Fields size(b, e);
    Triplets t;
    gidx nrows = 0, ncols = 0;
    auto push = [&](gidx r, gidx c, double re, double im) {
        t.push(r, c, re, im);
        if (r == c) {
            SK_REQUIRE(h.sym != MmSym::skew, errc::io, "skew-symmetric files must not contain diagonal entries");
            return;
        }
        switch (h.sym) {
            case MmSym::general: break;
            case MmSym::symmetric: t.push(c, r, re, im); break;
            case MmSym::skew: t.push(c, r, -re, -im); break;
            case MmSym::hermitian: t.push(c, r, re, -im); break;
        }
    };
    if (h.coordinate) {
        gidx nnz = 0;
        SK_REQUIRE(size.integer(nrows) && size.integer(ncols) && size.integer(nnz), errc::io, "malformed size line");
        if (nnz > 0) {
            t.row.reserve(std::size_t(nnz) * 2);
            t.col.reserve(std::size_t(nnz) * 2);
            t.re.reserve(std::size_t(nnz) * 2);
            t.im.reserve(std::size_t(nnz) * 2);
        }
        for (gidx k = 0; k < nnz; ++k) {
            SK_REQUIRE(lines.content(b, e), errc::io, "unexpected end of entries");
            Fields f(b, e);
            gidx i1 = 0, j1 = 0;
            double re = 1.0, im = 0.0;  // pattern entries are 1
            bool ok = f.integer(i1) && f.integer(j1);
            if (ok && h.field == MmField::complex_) ok = f.real(re) && f.real(im);
            else if (ok && h.field != MmField::pattern) ok = f.real(re);
            SK_REQUIRE(ok, errc::io, "malformed entry line");
            push(i1 - 1, j1 - 1, re, im);
        }
    } else {
        SK_REQUIRE(size.integer(nrows) && size.integer(ncols), errc::io, "malformed size line");
        const bool lower_only = h.sym != MmSym::general;
        if (lower_only) SK_REQUIRE(nrows == ncols, errc::io, "symmetric array matrices must be square");
        for (gidx j = 0; j < ncols; ++j) {
            const gidx i0 = lower_only ? (h.sym == MmSym::skew ? j + 1 : j) : 0;
            for (gidx i = i0; i < nrows; ++i) {
                SK_REQUIRE(lines.content(b, e), errc::io, "unexpected end of entries");
                Fields f(b, e);
                double re = 0.0, im = 0.0;
                bool ok = f.real(re);
                if (ok && h.field == MmField::complex_) ok = f.real(im);
                SK_REQUIRE(ok, errc::io, "malformed entry line");
                push(i, j, re, im);
            }
        }
    }
    return assemble(nrows, ncols, t, dt);
}

std::unique_ptr<Crs> crs_read_bin(const char* path) {
    const std::string bytes = slurp(path);
    Reader rd(bytes);
    rd.need(4);
    SK_REQUIRE(std::memcmp(bytes.data(), kMagic, 4) == 0, errc::io, "bad magic, not a binary CRS file");
    rd.pos = 4;
    SK_REQUIRE(rd.u32() == kVersion, errc::io, "unknown binary CRS version");
    const std::uint32_t flags = rd.u32();
    const std::uint64_t nrows = rd.u64(), ncols = rd.u64(), nnz = rd.u64();
    const bool cplx = flags & 1u, single = flags & 2u, wide = flags & 4u;
    const Datatype dt = cplx ? (single ? Datatype::c32 : Datatype::c64) : (single ? Datatype::r32 : Datatype::r64);
    SK_REQUIRE(nrows < (std::uint64_t(1) << 62) && ncols < (std::uint64_t(1) << 62) && nnz < (std::uint64_t(1) << 62),
               errc::io, "binary CRS dimensions out of range");
    // the whole payload must be present before anything is allocated from the header
    const std::size_t vb = value_bytes(dt);
    const std::uint64_t need = (nrows + 1) * 8 + nnz * (wide ? 8 : 4) + nnz * vb;
    SK_REQUIRE(std::uint64_t(bytes.size() - rd.pos) >= need, errc::io, "truncated binary CRS file");
    std::vector<gidx> rowptr(std::size_t(nrows) + 1);
    for (auto& p : rowptr) p = gidx(rd.u64());
    SK_REQUIRE(rowptr.front() == 0 && rowptr.back() == gidx(nnz), errc::io,
               "row pointer array inconsistent with header nonzero count");
    for (std::size_t r = 0; r + 1 < rowptr.size(); ++r)
        SK_REQUIRE(rowptr[r] <= rowptr[r + 1], errc::io, "row pointers must be non-decreasing");
    std::vector<gidx> col(static_cast<std::size_t>(nnz));
    if (wide)
        for (auto& c : col) c = gidx(rd.u64());
    else
        for (auto& c : col) c = gidx(rd.u32());
    rd.need(std::size_t(nnz) * vb);
    std::vector<unsigned char> val(bytes.begin() + std::ptrdiff_t(rd.pos),
                                   bytes.begin() + std::ptrdiff_t(rd.pos + std::size_t(nnz) * vb));
    rd.pos += std::size_t(nnz) * vb;
    SK_REQUIRE(rd.pos == bytes.size(), errc::io, "trailing bytes after binary CRS payload");
    return crs_from_host(dt, gidx(nrows), gidx(ncols), rowptr.data(), col.data(), val.data());
}

void crs_write_bin(const char* path, const Crs& a, bool wide_cols) {
    SK_REQUIRE(path != nullptr, errc::invalid_arg, "null path");
    crs_validate(a);
    std::vector<gidx> rowptr, col;
    std::vector<unsigned char> val;
    crs_download(a, rowptr, col, val);
    const bool wide = wide_cols || a.ncols > gidx(std::numeric_limits<std::int32_t>::max());
    std::string o;
    o.reserve(40 + rowptr.size() * 8 + col.size() * (wide ? 8 : 4) + val.size());
    o.append(kMagic, 4);
    put32(o, kVersion);
    std::uint32_t flags = 0;
    if (is_complex(a.dt)) flags |= 1u;
    if (a.dt == Datatype::r32 || a.dt == Datatype::c32) flags |= 2u;
    if (wide) flags |= 4u;
    put32(o, flags);
    put64(o, std::uint64_t(a.nrows));
    put64(o, std::uint64_t(a.ncols));
    put64(o, std::uint64_t(a.nnz));
    for (gidx p : rowptr) put64(o, std::uint64_t(p));
    if (wide)
        for (gidx c : col) put64(o, std::uint64_t(c));
    else
        for (gidx c : col) put32(o, std::uint32_t(c));
    o.append(reinterpret_cast<const char*>(val.data()), val.size());  // little-endian host
    FILE* f = std::fopen(path, "wb");
    SK_REQUIRE(f != nullptr, errc::io, std::string("cannot write ") + path);
    const std::size_t w = std::fwrite(o.data(), 1, o.size(), f);
    const int c = std::fclose(f);
    SK_REQUIRE(w == o.size() && c == 0, errc::io, std::string("write failure on ") + path);
}

}  // namespace skb
