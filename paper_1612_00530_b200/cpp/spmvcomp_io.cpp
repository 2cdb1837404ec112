// Binary serialization of the matrix and of the three formats, and Matrix Market export / import
// (include/spmvcomp/io.hpp, inc/stencil.hpp:61-64).  Host-only code: files either side of the
// device path.  The layout is written out in io.hpp.
#include "spmvcomp/io.hpp"

#include <algorithm>
#include <bit>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <type_traits>

namespace spmvcomp {
namespace {

static_assert(std::endian::native == std::endian::little, "the file layout is little-endian and written from memory as is");

constexpr char kMagic[8] = {'S', 'P', 'M', 'V', 'C', 'O', 'M', 'P'};

const char* kind_name(FileKind k) {
    switch (k) {
        case FileKind::stencil: return "StencilMatrix";
        case FileKind::ell: return "EllMatrix";
        case FileKind::vt: return "VtCompressedMatrix";
        case FileKind::pattern: return "PatternCompressedMatrix";
    }
    return "unknown";
}

// ---- sizes ----------------------------------------------------------------------------
template <class T>
std::uint64_t vec_bytes(const std::vector<T>& v) {
    return 8 + (std::uint64_t)v.size() * sizeof(T);
}
constexpr std::uint64_t kHeaderBytes = 16;

std::vector<std::int32_t> row_ends_of(const PatternCompressedMatrix& a) {  // inc/compress.hpp:62-64
    const std::size_t m = (std::size_t)a.table.size();
    std::vector<std::int32_t> e((std::size_t)a.n * m);
    for (std::int32_t i = 0; i < a.n; i++) {
        const std::int32_t id = a.row_pattern[(std::size_t)i];
        if (id < 0 || (std::size_t)id >= a.patterns.size() || a.patterns[(std::size_t)id].ends.size() != m)
            throw IntegrityError("save: row " + std::to_string(i) + " has pattern id " + std::to_string(id) + " without a matching table entry");
        std::copy(a.patterns[(std::size_t)id].ends.begin(), a.patterns[(std::size_t)id].ends.end(), e.begin() + (std::ptrdiff_t)((std::size_t)i * m));
    }
    return e;
}

// ---- writer ---------------------------------------------------------------------------
class Writer {
public:
    Writer(const std::filesystem::path& path, FileKind kind) : path_(path), out_(path, std::ios::binary | std::ios::trunc) {
        if (!out_) throw IoError("cannot open " + path.string() + " for writing");
        raw(kMagic, 8);
        scalar<std::uint32_t>(kFileVersion);
        scalar<std::uint32_t>((std::uint32_t)kind);
    }
    template <class T>
    void scalar(T v) {
        static_assert(std::is_trivially_copyable_v<T>);
        raw(&v, sizeof(T));
    }
    template <class T>
    void vec(const std::vector<T>& v) {
        scalar<std::uint64_t>(v.size());
        raw(v.data(), v.size() * sizeof(T));
    }
    void finish() {
        out_.flush();
        if (!out_) throw IoError("write to " + path_.string() + " failed");
    }

private:
    void raw(const void* p, std::size_t n) {
        if (n) out_.write(static_cast<const char*>(p), (std::streamsize)n);
        if (!out_) throw IoError("write to " + path_.string() + " failed");
    }
    std::filesystem::path path_;
    std::ofstream out_;
};

// ---- reader ---------------------------------------------------------------------------
class Reader {
public:
    explicit Reader(const std::filesystem::path& path) : path_(path), in_(path, std::ios::binary) {
        if (!in_) throw IoError("cannot open " + path.string());
        std::error_code ec;
        const auto sz = std::filesystem::file_size(path, ec);
        if (ec) throw IoError("cannot size " + path.string() + ": " + ec.message());
        left_ = sz;
        char magic[8];
        raw(magic, 8, "header");
        if (std::memcmp(magic, kMagic, 8) != 0) throw IoError(path.string() + ": not a spmvcomp file (bad magic)");
        const auto version = scalar<std::uint32_t>("version");
        if (version != kFileVersion) throw IoError(path.string() + ": unsupported file version " + std::to_string(version));
        const auto kind = scalar<std::uint32_t>("kind");
        if (kind < 1 || kind > 4) throw IoError(path.string() + ": unknown structure kind " + std::to_string(kind));
        kind_ = (FileKind)kind;
    }
    FileKind kind() const { return kind_; }
    void expect(FileKind k) const {
        if (kind_ != k) throw IoError(path_.string() + ": holds a " + kind_name(kind_) + ", not a " + kind_name(k));
    }
    template <class T>
    T scalar(const char* what) {
        T v;
        raw(&v, sizeof(T), what);
        return v;
    }
    template <class T>
    std::vector<T> vec(const char* what) {
        const auto count = scalar<std::uint64_t>(what);
        if (count > left_ / sizeof(T)) throw IoError(path_.string() + ": truncated in " + what + " (" + std::to_string(count) + " elements announced)");
        std::vector<T> v((std::size_t)count);
        raw(v.data(), (std::size_t)count * sizeof(T), what);
        return v;
    }
    bool flag(const char* what) {
        const auto b = scalar<std::uint8_t>(what);
        if (b > 1) throw IoError(path_.string() + ": " + what + " is not 0 or 1");
        return b == 1;
    }
    void finish() const {
        if (left_ != 0) throw IoError(path_.string() + ": " + std::to_string(left_) + " trailing bytes");
    }
    [[noreturn]] void bad(const std::string& why) const { throw IoError(path_.string() + ": " + why); }

private:
    void raw(void* p, std::size_t n, const char* what) {
        if (n > left_) throw IoError(path_.string() + ": truncated in " + what);
        if (n) in_.read(static_cast<char*>(p), (std::streamsize)n);
        if (!in_) throw IoError(path_.string() + ": read failed in " + what);
        left_ -= n;
    }
    std::filesystem::path path_;
    std::ifstream in_;
    std::uint64_t left_ = 0;
    FileKind kind_ = FileKind::stencil;
};

}  // namespace

// ---- sizes ------------------------------------------------------------------------------
std::uint64_t serialized_size(const StencilMatrix& m) {
    return kHeaderBytes + 4 + vec_bytes(m.row_start) + vec_bytes(m.cols) + vec_bytes(m.vals) + 12;
}
std::uint64_t serialized_size(const EllMatrix& a) { return kHeaderBytes + 4 + 4 + 8 + vec_bytes(a.values) + vec_bytes(a.columns); }
std::uint64_t serialized_size(const VtCompressedMatrix& a) {
    return kHeaderBytes + 4 + 4 + vec_bytes(a.table.entries) + vec_bytes(a.sorted_columns) + vec_bytes(a.ends);
}
std::uint64_t serialized_size(const PatternCompressedMatrix& a) {
    std::uint64_t b = kHeaderBytes + 4 + vec_bytes(a.table.entries) + 8;
    for (const auto& p : a.patterns) b += vec_bytes(p.displacements) + vec_bytes(p.ends);
    b += vec_bytes(a.row_pattern) + 1;
    if (!a.values_in_pattern) b += 8 + (std::uint64_t)a.n * (std::uint64_t)a.table.size() * 4;
    return b;
}

// ---- save -------------------------------------------------------------------------------
void save(const StencilMatrix& m, const std::filesystem::path& path) {
    Writer w(path, FileKind::stencil);
    w.scalar<std::int32_t>(m.n);
    w.vec(m.row_start);
    w.vec(m.cols);
    w.vec(m.vals);
    w.scalar<std::int32_t>(m.grid.nx);
    w.scalar<std::int32_t>(m.grid.ny);
    w.scalar<std::int32_t>(m.grid.nz);
    w.finish();
}

void save(const EllMatrix& a, const std::filesystem::path& path) {
    Writer w(path, FileKind::ell);
    w.scalar<std::int32_t>(a.n);
    w.scalar<std::int32_t>(a.width);
    w.scalar<std::int64_t>(a.nnz);
    w.vec(a.values);
    w.vec(a.columns);
    w.finish();
}

void save(const VtCompressedMatrix& a, const std::filesystem::path& path) {
    Writer w(path, FileKind::vt);
    w.scalar<std::int32_t>(a.n);
    w.scalar<std::int32_t>(a.width);
    w.vec(a.table.entries);
    w.vec(a.sorted_columns);
    w.vec(a.ends);
    w.finish();
}

void save(const PatternCompressedMatrix& a, const std::filesystem::path& path) {
    std::vector<std::int32_t> row_ends;
    if (!a.values_in_pattern) row_ends = row_ends_of(a);  // before the file is touched: may throw IntegrityError
    Writer w(path, FileKind::pattern);
    w.scalar<std::int32_t>(a.n);
    w.vec(a.table.entries);
    w.scalar<std::uint64_t>(a.patterns.size());
    for (const auto& p : a.patterns) {
        w.vec(p.displacements);
        w.vec(p.ends);
    }
    w.vec(a.row_pattern);
    w.scalar<std::uint8_t>(a.values_in_pattern ? 1 : 0);
    if (!a.values_in_pattern) w.vec(row_ends);
    w.finish();
}

// ---- load -------------------------------------------------------------------------------
FileKind file_kind(const std::filesystem::path& path) { return Reader(path).kind(); }

StencilMatrix load_stencil(const std::filesystem::path& path) {
    Reader r(path);
    r.expect(FileKind::stencil);
    StencilMatrix m;
    m.n = r.scalar<std::int32_t>("n");
    m.row_start = r.vec<std::int64_t>("row_start");
    m.cols = r.vec<std::int32_t>("cols");
    m.vals = r.vec<double>("vals");
    m.grid.nx = r.scalar<std::int32_t>("grid.nx");
    m.grid.ny = r.scalar<std::int32_t>("grid.ny");
    m.grid.nz = r.scalar<std::int32_t>("grid.nz");
    r.finish();
    if (m.n < 0 || m.row_start.size() != (std::size_t)m.n + 1) r.bad("row_start does not have n + 1 entries");
    if (m.row_start.front() != 0 || !std::is_sorted(m.row_start.begin(), m.row_start.end())) r.bad("row_start is not a non-decreasing sequence from 0");
    if ((std::uint64_t)m.row_start.back() != m.cols.size() || m.cols.size() != m.vals.size()) r.bad("cols / vals do not have row_start[n] entries");
    return m;
}

EllMatrix load_ell(const std::filesystem::path& path) {
    Reader r(path);
    r.expect(FileKind::ell);
    EllMatrix a;
    a.n = r.scalar<std::int32_t>("n");
    a.width = r.scalar<std::int32_t>("width");
    a.nnz = r.scalar<std::int64_t>("nnz");
    a.values = r.vec<double>("values");
    a.columns = r.vec<std::int32_t>("columns");
    r.finish();
    const std::uint64_t slots = (std::uint64_t)std::max(a.n, 0) * (std::uint64_t)std::max(a.width, 0);
    if (a.n < 0 || a.width < 0 || a.values.size() != slots || a.columns.size() != slots) r.bad("values / columns do not have n * width entries");
    if (a.nnz < 0 || (std::uint64_t)a.nnz > slots) r.bad("nnz exceeds n * width");
    return a;
}

VtCompressedMatrix load_vt(const std::filesystem::path& path) {
    Reader r(path);
    r.expect(FileKind::vt);
    VtCompressedMatrix a;
    a.n = r.scalar<std::int32_t>("n");
    a.width = r.scalar<std::int32_t>("width");
    a.table.entries = r.vec<double>("table");
    a.sorted_columns = r.vec<std::int32_t>("sorted_columns");
    a.ends = r.vec<std::int32_t>("ends");
    r.finish();
    if (a.n < 0 || a.width < 0) r.bad("negative n or width");
    if (a.sorted_columns.size() != (std::uint64_t)a.n * (std::uint64_t)a.width) r.bad("sorted_columns does not have n * width entries");
    if (a.ends.size() != (std::uint64_t)a.n * a.table.entries.size()) r.bad("ends does not have n * table.size() entries");
    return a;
}

PatternCompressedMatrix load_pattern(const std::filesystem::path& path) {
    Reader r(path);
    r.expect(FileKind::pattern);
    PatternCompressedMatrix a;
    a.n = r.scalar<std::int32_t>("n");
    a.table.entries = r.vec<double>("table");
    const auto n_patterns = r.scalar<std::uint64_t>("pattern count");
    if (n_patterns > (std::uint64_t)INT32_MAX) r.bad("pattern count does not fit a pattern id");
    for (std::uint64_t p = 0; p < n_patterns; p++) {
        DisplacementPattern dp;
        dp.displacements = r.vec<std::int32_t>("displacements");
        dp.ends = r.vec<std::int32_t>("pattern ends");
        if (dp.ends.size() != a.table.entries.size()) r.bad("pattern " + std::to_string(p) + " does not have table.size() ends");
        a.patterns.push_back(std::move(dp));
    }
    a.row_pattern = r.vec<std::int32_t>("row_pattern");
    a.values_in_pattern = r.flag("values_in_pattern");
    std::vector<std::int32_t> row_ends;
    if (!a.values_in_pattern) row_ends = r.vec<std::int32_t>("per-row ends");
    r.finish();
    if (a.n < 0 || a.row_pattern.size() != (std::size_t)a.n) r.bad("row_pattern does not have n entries");
    if (!a.values_in_pattern) {
        const std::size_t m = a.table.entries.size();
        if (row_ends.size() != (std::uint64_t)a.n * m) r.bad("per-row ends do not have n * table.size() entries");
        for (std::int32_t i = 0; i < a.n; i++) {
            const std::int32_t id = a.row_pattern[(std::size_t)i];
            if (id < 0 || (std::uint64_t)id >= n_patterns ||
                !std::equal(a.patterns[(std::size_t)id].ends.begin(), a.patterns[(std::size_t)id].ends.end(), row_ends.begin() + (std::ptrdiff_t)((std::size_t)i * m)))
                throw IntegrityError(path.string() + ": per-row ends of row " + std::to_string(i) + " disagree with the pattern table");
        }
    }
    return a;
}

// ---- Matrix Market ------------------------------------------------------------------------
void write_matrix_market(const StencilMatrix& m, const std::filesystem::path& path) {
    if (!is_symmetric(m)) throw std::invalid_argument("write_matrix_market: the matrix is not symmetric");
    std::int64_t lower = 0;
    for (std::int32_t i = 0; i < m.n; i++)
        for (const std::int32_t c : m.row_cols(i)) lower += c <= i;
    std::FILE* f = std::fopen(path.string().c_str(), "w");
    if (!f) throw IoError("cannot open " + path.string() + " for writing");
    bool ok = std::fprintf(f, "%%%%MatrixMarket matrix coordinate real symmetric\n%d %d %" PRId64 "\n", m.n, m.n, lower) > 0;
    for (std::int32_t i = 0; i < m.n && ok; i++) {
        const auto cols = m.row_cols(i);
        const auto vals = m.row_vals(i);
        for (std::size_t t = 0; t < cols.size() && cols[t] <= i && ok; t++) ok = std::fprintf(f, "%d %d %.17g\n", i + 1, cols[t] + 1, vals[t]) > 0;
    }
    ok = std::fclose(f) == 0 && ok;
    if (!ok) throw IoError("write to " + path.string() + " failed");
}

StencilMatrix read_matrix_market(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open " + path.string());
    std::string line;
    if (!std::getline(in, line)) throw IoError(path.string() + ": empty file");
    std::istringstream banner(line);
    std::string tag, object, format, field, symmetry;
    banner >> tag >> object >> format >> field >> symmetry;
    if (tag != "%%MatrixMarket" || object != "matrix" || format != "coordinate" || field != "real" || (symmetry != "symmetric" && symmetry != "general"))
        throw IoError(path.string() + ": only 'matrix coordinate real symmetric|general' files are read");
    while (std::getline(in, line) && (line.empty() || line[0] == '%')) {}
    long long rows = 0, cols = 0, entries = 0;
    if (std::sscanf(line.c_str(), "%lld %lld %lld", &rows, &cols, &entries) != 3 || rows < 0 || rows != cols || rows > INT32_MAX || entries < 0)
        throw IoError(path.string() + ": bad size line");
    std::vector<std::vector<std::pair<std::int32_t, double>>> by_row((std::size_t)rows);
    for (long long e = 0; e < entries; e++) {
        long long i = 0, j = 0;
        double v = 0.0;
        if (!(in >> i >> j >> v) || i < 1 || j < 1 || i > rows || j > rows) throw IoError(path.string() + ": bad or missing entry " + std::to_string(e + 1));
        by_row[(std::size_t)(i - 1)].emplace_back((std::int32_t)(j - 1), v);
        if (symmetry == "symmetric" && i != j) by_row[(std::size_t)(j - 1)].emplace_back((std::int32_t)(i - 1), v);
    }
    // rows in ascending column order (inc/stencil.hpp:15-16); built on the host: no device is involved in reading a file
    StencilMatrix m;
    m.n = (std::int32_t)rows;
    m.row_start.assign(1, 0);
    for (auto& r : by_row) {
        std::sort(r.begin(), r.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        for (std::size_t t = 0; t < r.size(); t++) {
            if (t > 0 && r[t].first == r[t - 1].first) throw IoError(path.string() + ": duplicate entry");
            m.cols.push_back(r[t].first);
            m.vals.push_back(r[t].second);
        }
        m.row_start.push_back((std::int64_t)m.cols.size());
    }
    return m;
}

}  // namespace spmvcomp
