// Host-side C++ implementation of the spmvcomp API (include/spmvcomp/spmvcomp.hpp) on top
// of the C-ABI (include/spmvcomp_b200.h).  Every operation runs on the GPU: host structs are
// uploaded, the device kernel / builder runs, results are copied back.  A failed C-ABI call
// becomes the reference exception its status code stands for.  There is no CPU fallback.
//
// This file also compiles against the reference's own headers
// (g++ -I/root/reference/proj/include ...), which is how tests/test_cpp_api.py checks that
// the signatures are drop-in compatible.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>

#include "spmvcomp/compress.hpp"
#include "spmvcomp/ell.hpp"
#include "spmvcomp/errors.hpp"
#include "spmvcomp/grid.hpp"
#include "spmvcomp/kernels.hpp"
#include "spmvcomp/perf_model.hpp"
#include "spmvcomp/solver.hpp"
#include "spmvcomp/stencil.hpp"
#include "spmvcomp_b200/device.hpp"

namespace spmvcomp {
namespace b200 {

void throw_on_error(int status) {
    if (status == SPMVB_OK) return;
    const std::string msg = spmvb_last_error();
    switch (status) {
        case SPMVB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SPMVB_ERR_TABLE_OVERFLOW: throw TableOverflowError(msg);
        case SPMVB_ERR_INTEGRITY: throw IntegrityError(msg);
        case SPMVB_ERR_VERIFICATION: throw VerificationError(msg);
        case SPMVB_ERR_IO: throw IoError(msg);
        case SPMVB_ERR_DIVERGENCE: throw DivergenceError(-1, msg);
        case SPMVB_ERR_NOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);  // CUDA / NCCL
    }
}

namespace {

template <class T>
std::vector<T> pull(const spmvb_matrix* h, int sid) {
    uint64_t bytes = 0;
    throw_on_error(spmvb_matrix_stream_bytes(h, sid, &bytes));
    std::vector<T> out(bytes / sizeof(T));
    throw_on_error(spmvb_matrix_download(h, sid, 0, bytes, out.data()));
    return out;
}

spmvb_compress_options copts(const CompressOptions& o, bool vip, int min_rows, int cap) {
    spmvb_compress_options c{};
    c.value_table_limit = o.value_table_limit;
    c.values_in_pattern = vip;
    c.min_pattern_rows = min_rows;
    c.dict_cap = cap;
    return c;
}

}  // namespace

DeviceMatrix& DeviceMatrix::operator=(DeviceMatrix&& o) noexcept {
    if (this != &o) {
        if (h_) spmvb_matrix_destroy(h_);
        h_ = o.h_;
        o.h_ = nullptr;
    }
    return *this;
}
DeviceMatrix::~DeviceMatrix() {
    if (h_) spmvb_matrix_destroy(h_);
}
DeviceMatrix::DeviceMatrix(const StencilMatrix& m) {
    if ((std::int64_t)m.row_start.size() != (std::int64_t)m.n + 1) throw std::invalid_argument("StencilMatrix: row_start must hold n+1 offsets");
    throw_on_error(spmvb_csr_upload(m.n, m.n, 0, m.row_start.data(), m.cols.data(), m.vals.data(), &h_));
}
DeviceMatrix::DeviceMatrix(const EllMatrix& a) {
    if ((std::int64_t)a.values.size() != a.slot(a.n, 0) || a.columns.size() != a.values.size())
        throw std::invalid_argument("EllMatrix: values/columns must hold n*width entries");
    throw_on_error(spmvb_ell_upload(a.n, a.width, a.nnz, 0, a.values.data(), a.columns.data(), &h_));
}
DeviceMatrix::DeviceMatrix(const VtCompressedMatrix& a) {
    const std::int64_t m = a.table.size();
    if ((std::int64_t)a.sorted_columns.size() != (std::int64_t)a.n * a.width || (std::int64_t)a.ends.size() != (std::int64_t)a.n * m)
        throw std::invalid_argument("VtCompressedMatrix: array sizes do not match n, width and the table");
    throw_on_error(spmvb_vt_upload(a.n, a.width, (int32_t)m, 0, a.table.entries.data(), a.sorted_columns.data(), a.ends.data(), &h_));
}
DeviceMatrix::DeviceMatrix(const PatternCompressedMatrix& a) {
    const std::int32_t m = a.table.size();
    if ((std::int64_t)a.row_pattern.size() != a.n) throw std::invalid_argument("PatternCompressedMatrix: row_pattern must hold n ids");
    std::vector<std::int64_t> off(a.patterns.size() + 1, 0);
    std::vector<std::int32_t> disp, ends;
    for (std::size_t p = 0; p < a.patterns.size(); p++) {
        if ((std::int32_t)a.patterns[p].ends.size() != m) throw IntegrityError("pattern " + std::to_string(p) + ": ends must hold one entry per table value");
        disp.insert(disp.end(), a.patterns[p].displacements.begin(), a.patterns[p].displacements.end());
        ends.insert(ends.end(), a.patterns[p].ends.begin(), a.patterns[p].ends.end());
        off[p + 1] = (std::int64_t)disp.size();
    }
    for (std::int32_t id : a.row_pattern)  // the reference format has no exception rows: every id must be valid
        if (id < 0 || id >= (std::int32_t)a.patterns.size()) throw IntegrityError("pattern id " + std::to_string(id) + " out of range");
    throw_on_error(spmvb_pattern_upload(a.n, m, 0, a.table.entries.data(), (int32_t)a.patterns.size(), off.data(), disp.data(),
                                        ends.data(), a.row_pattern.data(), a.values_in_pattern, 0, 0, nullptr, nullptr, nullptr, &h_));
}

spmvb_matrix_info DeviceMatrix::info() const {
    spmvb_matrix_info i{};
    throw_on_error(spmvb_matrix_get_info(h_, &i));
    return i;
}

DeviceMatrix DeviceMatrix::generate(const GridSpec& spec, double diagonal, double off_diagonal, std::int64_t row_begin,
                                    std::int64_t row_end) {
    validate(spec);
    spmvb_grid g{};
    g.nx = spec.nx; g.ny = spec.ny; g.nz = spec.nz;
    g.diagonal = diagonal; g.off_diagonal = off_diagonal;
    spmvb_matrix* h = nullptr;
    throw_on_error(spmvb_generate_csr(&g, row_begin, row_end < 0 ? spec.rows() : row_end, nullptr, &h));
    return DeviceMatrix(h);
}
DeviceMatrix DeviceMatrix::to_ell(std::int32_t min_width) const {
    spmvb_matrix* h = nullptr;
    throw_on_error(spmvb_csr_to_ell(h_, min_width, nullptr, &h));
    return DeviceMatrix(h);
}
DeviceMatrix DeviceMatrix::compress_values(const CompressOptions& o, std::int32_t min_width) const {
    spmvb_matrix* h = nullptr;
    const spmvb_compress_options c = copts(o, false, 1, 0);
    throw_on_error(spmvb_csr_compress_values(h_, &c, min_width, nullptr, &h));
    return DeviceMatrix(h);
}
DeviceMatrix DeviceMatrix::compress_patterns(bool vip, const CompressOptions& o) const {
    spmvb_matrix* h = nullptr;
    const spmvb_compress_options c = copts(o, vip, 1, 0);
    throw_on_error(spmvb_csr_compress_patterns(h_, &c, nullptr, &h));
    return DeviceMatrix(h);
}
DeviceMatrix DeviceMatrix::compress_hybrid(bool vip, const HybridOptions& hy, const CompressOptions& o) const {
    spmvb_matrix* h = nullptr;
    const spmvb_compress_options c = copts(o, vip, hy.min_pattern_rows, hy.dict_cap);
    throw_on_error(spmvb_csr_compress_patterns(h_, &c, nullptr, &h));
    return DeviceMatrix(h);
}
DeviceMatrix DeviceMatrix::to_csr() const {
    spmvb_matrix* h = nullptr;
    throw_on_error(spmvb_to_csr(h_, nullptr, &h));
    return DeviceMatrix(h);
}

StencilMatrix DeviceMatrix::download_csr() const {
    const spmvb_matrix_info i = info();
    if (i.format != SPMVB_FMT_CSR) throw std::invalid_argument("download_csr: handle is not a CSR matrix");
    StencilMatrix m;
    m.n = i.n;
    m.row_start = pull<std::int64_t>(h_, SPMVB_S_CSR_ROW_START);
    m.cols = pull<std::int32_t>(h_, SPMVB_S_CSR_COLS);
    m.vals = pull<double>(h_, SPMVB_S_CSR_VALS);
    return m;
}
EllMatrix DeviceMatrix::download_ell() const {
    const spmvb_matrix_info i = info();
    if (i.format != SPMVB_FMT_ELL) throw std::invalid_argument("download_ell: handle is not an ELL matrix");
    EllMatrix a;
    a.n = i.n; a.width = i.width; a.nnz = i.nnz;
    a.values = pull<double>(h_, SPMVB_S_VALUES);
    a.columns = pull<std::int32_t>(h_, SPMVB_S_COLUMNS);
    return a;
}
VtCompressedMatrix DeviceMatrix::download_vt() const {
    const spmvb_matrix_info i = info();
    if (i.format != SPMVB_FMT_VT) throw std::invalid_argument("download_vt: handle is not a value-table matrix");
    VtCompressedMatrix a;
    a.n = i.n; a.width = i.width;
    a.table.entries = pull<double>(h_, SPMVB_S_TABLE);
    a.sorted_columns = pull<std::int32_t>(h_, SPMVB_S_SORTED_COLUMNS);
    a.ends = pull<std::int32_t>(h_, SPMVB_S_ENDS);
    return a;
}
PatternCompressedMatrix DeviceMatrix::download_pattern() const {
    const spmvb_matrix_info i = info();
    if (i.format != SPMVB_FMT_PATTERN) throw std::invalid_argument("download_pattern: handle is not a pattern matrix");
    if (i.n_exc != 0) throw std::invalid_argument("download_pattern: exception rows do not fit PatternCompressedMatrix");
    PatternCompressedMatrix a;
    a.n = i.n;
    a.values_in_pattern = i.values_in_pattern != 0;
    a.table.entries = pull<double>(h_, SPMVB_S_TABLE);
    a.row_pattern = pull<std::int32_t>(h_, SPMVB_S_ROW_PATTERN);
    const auto off = pull<std::int64_t>(h_, SPMVB_S_DISP_OFFSETS);
    const auto disp = pull<std::int32_t>(h_, SPMVB_S_DISP_FLAT);
    const auto ends = pull<std::int32_t>(h_, SPMVB_S_ENDS_FLAT);
    a.patterns.resize(i.n_patterns);
    for (int p = 0; p < i.n_patterns; p++) {
        a.patterns[p].displacements.assign(disp.begin() + off[p], disp.begin() + off[p + 1]);
        a.patterns[p].ends.assign(ends.begin() + (std::ptrdiff_t)p * i.m, ends.begin() + (std::ptrdiff_t)(p + 1) * i.m);
    }
    return a;
}

DeviceVector::DeviceVector(std::int64_t n) : n_(n) { throw_on_error(spmvb_vec_alloc(n, &p_)); }
DeviceVector::DeviceVector(std::span<const double> host) : n_((std::int64_t)host.size()) {
    throw_on_error(spmvb_vec_alloc(n_, &p_));
    upload(host);
}
DeviceVector::~DeviceVector() {
    if (p_) spmvb_vec_free(p_);
}
void DeviceVector::upload(std::span<const double> host) {
    if ((std::int64_t)host.size() != n_) throw std::invalid_argument("DeviceVector::upload: length mismatch");
    throw_on_error(spmvb_vec_upload(p_, host.data(), n_, nullptr));
}
Vector DeviceVector::download() const {
    Vector v((std::size_t)n_);
    throw_on_error(spmvb_vec_download(v.data(), p_, n_, nullptr));
    return v;
}
void DeviceVector::fill(VectorKind kind, std::uint64_t seed, double lo, double hi, std::int64_t first_index) {
    throw_on_error(spmvb_vec_fill(p_, n_, (int32_t)kind, seed, lo, hi, first_index, nullptr));
}

void spmv_rows(const DeviceMatrix& a, const DeviceVector& x, DeviceVector& y, std::int32_t begin, std::int32_t end, void* stream) {
    throw_on_error(spmvb_spmv(a.handle(), x.data(), 0, x.size(), y.data(), begin, end, stream));
}

}  // namespace b200

using b200::DeviceMatrix;
using b200::throw_on_error;

// ---------------------------------------------------------------- equality (bit patterns for values)
namespace {
bool same_doubles(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && (a.empty() || !std::memcmp(a.data(), b.data(), a.size() * sizeof(double)));
}
}  // namespace

bool operator==(const StencilMatrix& a, const StencilMatrix& b) {
    return a.n == b.n && a.row_start == b.row_start && a.cols == b.cols && same_doubles(a.vals, b.vals);
}
bool operator==(const EllMatrix& a, const EllMatrix& b) {
    return a.n == b.n && a.width == b.width && a.nnz == b.nnz && a.columns == b.columns && same_doubles(a.values, b.values);
}
bool operator==(const VtCompressedMatrix& a, const VtCompressedMatrix& b) {
    return a.n == b.n && a.width == b.width && same_doubles(a.table.entries, b.table.entries) &&
           a.sorted_columns == b.sorted_columns && a.ends == b.ends;
}
bool operator==(const PatternCompressedMatrix& a, const PatternCompressedMatrix& b) {
    return a.n == b.n && same_doubles(a.table.entries, b.table.entries) && a.patterns == b.patterns &&
           a.row_pattern == b.row_pattern && a.values_in_pattern == b.values_in_pattern;
}

std::int64_t VtCompressedMatrix::nnz() const {
    std::int64_t s = 0;
    for (std::int32_t i = 0; i < n; i++) s += row_nnz(i);
    return s;
}
std::int64_t PatternCompressedMatrix::nnz() const {
    std::int64_t s = 0;
    for (std::int32_t i = 0; i < n; i++) s += row_nnz(i);
    return s;
}

// ---------------------------------------------------------------- generator and vectors
StencilMatrix generate_matrix(const GridSpec& spec, double diagonal, double off_diagonal) {
    StencilMatrix m = DeviceMatrix::generate(spec, diagonal, off_diagonal).download_csr();
    m.grid = spec;
    return m;
}

StencilMatrix stencil_from_rows(std::int32_t n, const std::vector<std::vector<std::pair<std::int32_t, double>>>& rows) {
    if (n < 0 || (std::int64_t)rows.size() != n) throw std::invalid_argument("stencil_from_rows: need exactly n rows");
    StencilMatrix m;
    m.n = n;
    m.row_start.assign(1, 0);
    for (const auto& r : rows) {
        for (const auto& [c, v] : r) {
            m.cols.push_back(c);
            m.vals.push_back(v);
        }
        m.row_start.push_back((std::int64_t)m.cols.size());
    }
    DeviceMatrix check(m);  // the C-ABI validates: strictly ascending, in-range columns
    return m;
}

bool is_symmetric(const StencilMatrix& m) {
    for (std::int32_t i = 0; i < m.n; i++) {
        const auto ci = m.row_cols(i);
        const auto vi = m.row_vals(i);
        for (std::size_t t = 0; t < ci.size(); t++) {
            const auto cj = m.row_cols(ci[t]);
            const auto it = std::lower_bound(cj.begin(), cj.end(), i);
            if (it == cj.end() || *it != i) return false;
            const double w = m.row_vals(ci[t])[(std::size_t)(it - cj.begin())];
            if (std::memcmp(&w, &vi[t], sizeof(double))) return false;
        }
    }
    return true;
}

Vector make_test_vector(std::int64_t n, VectorKind kind, std::optional<std::uint64_t> seed) {
    if (n < 1) throw std::invalid_argument("make_test_vector: n must be >= 1");
    if (kind == VectorKind::random && !seed) throw std::invalid_argument("make_test_vector: the random kind needs a seed");
    b200::DeviceVector v(n);
    v.fill(kind, seed.value_or(0), 0.0, 1.0, 0);
    return v.download();
}

// ---------------------------------------------------------------- formats
EllMatrix to_ell(const StencilMatrix& m) { return DeviceMatrix(m).to_ell().download_ell(); }
StencilMatrix to_stencil(const EllMatrix& a) { return DeviceMatrix(a).to_csr().download_csr(); }

ValueTable scan_value_table(const StencilMatrix& m, std::size_t limit) {
    CompressOptions o;
    o.value_table_limit = limit;
    return DeviceMatrix(m).compress_values(o).download_vt().table;
}
VtCompressedMatrix compress_values(const StencilMatrix& m, const CompressOptions& opts) {
    return DeviceMatrix(m).compress_values(opts).download_vt();
}
PatternCompressedMatrix compress_patterns(const StencilMatrix& m, bool values_in_pattern, const CompressOptions& opts) {
    return DeviceMatrix(m).compress_patterns(values_in_pattern, opts).download_pattern();
}
StencilMatrix decompress(const VtCompressedMatrix& c) { return DeviceMatrix(c).to_csr().download_csr(); }
StencilMatrix decompress(const PatternCompressedMatrix& c) { return DeviceMatrix(c).to_csr().download_csr(); }
void validate(const VtCompressedMatrix& c) {
    DeviceMatrix d(c);
    throw_on_error(spmvb_validate(d.handle(), c.n, nullptr));
}
void validate(const PatternCompressedMatrix& c) {
    DeviceMatrix d(c);
    throw_on_error(spmvb_validate(d.handle(), c.n, nullptr));
}

// ---------------------------------------------------------------- SpMV
namespace {
template <class Fmt>
Vector spmv_checked(const Fmt& a, const Vector& x, bool check) {
    DeviceMatrix d(a);
    if (check) throw_on_error(spmvb_validate(d.handle(), a.n, nullptr));
    Vector y((std::size_t)a.n);
    throw_on_error(spmvb_spmv_host(d.handle(), x.data(), (std::int64_t)x.size(), y.data()));  // length mismatch -> invalid_argument
    return y;
}
template <class Fmt>
void rows_impl(const Fmt& a, std::span<const double> x, std::span<double> y, std::int32_t begin, std::int32_t end) {
    if (end <= begin) return;
    DeviceMatrix d(a);
    b200::DeviceVector dx(x), dy((std::int64_t)y.size());
    throw_on_error(spmvb_spmv(d.handle(), dx.data(), 0, dx.size(), dy.data(), begin, end, nullptr));
    const Vector out = dy.download();
    std::copy(out.begin() + begin, out.begin() + end, y.begin() + begin);  // rows outside [begin,end) untouched
}
}  // namespace

Vector spmv(const EllMatrix& a, const Vector& x) { return spmv_checked(a, x, true); }  // inc/kernels.hpp:23: validated like the other two
Vector spmv(const VtCompressedMatrix& a, const Vector& x) { return spmv_checked(a, x, true); }
Vector spmv(const PatternCompressedMatrix& a, const Vector& x) { return spmv_checked(a, x, true); }

namespace unchecked {
void spmv_rows(const EllMatrix& a, std::span<const double> x, std::span<double> y, std::int32_t b, std::int32_t e) { rows_impl(a, x, y, b, e); }
void spmv_rows(const VtCompressedMatrix& a, std::span<const double> x, std::span<double> y, std::int32_t b, std::int32_t e) { rows_impl(a, x, y, b, e); }
void spmv_rows(const PatternCompressedMatrix& a, std::span<const double> x, std::span<double> y, std::int32_t b, std::int32_t e) { rows_impl(a, x, y, b, e); }
}  // namespace unchecked

// ---------------------------------------------------------------- CG caller
double dot(const Vector& u, const Vector& v) {
    if (u.size() != v.size()) throw std::invalid_argument("dot: length mismatch");
    if (u.empty()) return 0.0;
    b200::DeviceVector du(u), dv(v);
    double out = 0.0;
    throw_on_error(spmvb_dot(du.data(), dv.data(), du.size(), &out, nullptr));
    return out;
}
void waxpby_into(double alpha, const Vector& x, double beta, const Vector& y, Vector& w) {
    if (x.size() != y.size()) throw std::invalid_argument("waxpby: length mismatch");
    w.resize(x.size());
    if (x.empty()) return;
    b200::DeviceVector dx(x), dy(y), dw((std::int64_t)x.size());
    throw_on_error(spmvb_waxpby(alpha, dx.data(), beta, dy.data(), dw.data(), dx.size(), nullptr));
    w = dw.download();
}
Vector waxpby(double alpha, const Vector& x, double beta, const Vector& y) {
    Vector w;
    waxpby_into(alpha, x, beta, y, w);
    return w;
}
const char* backend_name(SpmvBackend b) {
    return b == SpmvBackend::ell ? "ell" : (b == SpmvBackend::vt ? "vt" : "pattern");
}
void symgs_sweep(const StencilMatrix& m, Vector& x, const Vector& b) {
    if ((std::int64_t)x.size() != m.n || (std::int64_t)b.size() != m.n) throw std::invalid_argument("symgs_sweep: x or b has the wrong length");
    if (m.grid.rows() != m.n) throw std::invalid_argument("symgs_sweep: the device sweep needs the matrix's grid (StencilMatrix::grid)");
    DeviceMatrix csr(m);
    b200::DeviceVector dx(x), db(b);
    spmvb_grid sg{};
    sg.nx = m.grid.nx, sg.ny = m.grid.ny, sg.nz = m.grid.nz;
    throw_on_error(spmvb_symgs_sweep(csr.handle(), &sg, dx.data(), db.data(), nullptr));
    x = dx.download();
}

std::pair<Vector, CgReport> cg_solve(const StencilMatrix& m, const Vector& b, const CgConfig& cfg) {
    if ((std::int64_t)b.size() != m.n) throw std::invalid_argument("cg_solve: b has the wrong length");
    if (cfg.max_iterations < 1 || !(cfg.tolerance > 0.0)) throw std::invalid_argument("cg_solve: need max_iterations >= 1 and tolerance > 0");
    if (cfg.symgs_sweeps < 0) throw std::invalid_argument("cg_solve: symgs_sweeps must be >= 0");
    if (cfg.symgs_sweeps > 0 && m.grid.rows() != m.n)
        throw std::invalid_argument("cg_solve: the SymGS preconditioner needs the matrix's grid (StencilMatrix::grid)");
    DeviceMatrix csr(m);
    DeviceMatrix a = cfg.backend == SpmvBackend::ell ? csr.to_ell()
                   : cfg.backend == SpmvBackend::vt ? csr.compress_values() : csr.compress_patterns(true);
    b200::DeviceVector db(b), dx(m.n);
    CgReport rep;
    rep.residual_history.assign((std::size_t)cfg.max_iterations + 1, 0.0);
    std::int32_t it = 0, conv = 0;
    const auto t0 = std::chrono::steady_clock::now();
    spmvb_grid sg{};
    sg.nx = m.grid.nx, sg.ny = m.grid.ny, sg.nz = m.grid.nz;
    const int rc = cfg.symgs_sweeps > 0
                       ? spmvb_pcg_solve(a.handle(), csr.handle(), &sg, cfg.symgs_sweeps, db.data(), dx.data(), cfg.max_iterations, cfg.tolerance,
                                         &it, &conv, rep.residual_history.data(), nullptr)
                       : spmvb_cg_solve(a.handle(), db.data(), dx.data(), cfg.max_iterations, cfg.tolerance, &it, &conv,
                                        rep.residual_history.data(), nullptr);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (rc == SPMVB_ERR_DIVERGENCE) throw DivergenceError(it, spmvb_last_error());
    throw_on_error(rc);
    rep.iterations = it;
    rep.converged = conv != 0;
    rep.residual_history.resize((std::size_t)it + 1);
    // inc/solver.hpp:43: per iteration 2*nnz (SpMV) + 3 dots (6n) + 3 waxpbys (6n)
    rep.per_op["spmv"] = {it, it * spmv_flops(m.nnz()), 0.0};
    rep.per_op["dot"] = {3LL * it, 3LL * it * dot_flops(m.n), 0.0};
    rep.per_op["waxpby"] = {3LL * it, 3LL * it * waxpby_flops(m.n), 0.0};
    // one application before the loop and one per iteration that goes on: symgs_flops per sweep (inc/kernels.hpp:17)
    const std::int64_t applications = cfg.symgs_sweeps > 0 ? (std::int64_t)it + (conv ? 0 : 1) : 0;
    rep.per_op["precond"] = {applications, applications * cfg.symgs_sweeps * symgs_flops(m.nnz()), 0.0};
    rep.per_op["spmv"].seconds = secs;  // the loop is timed as a whole on the device path
    rep.flops_total = rep.per_op["spmv"].flops + rep.per_op["dot"].flops + rep.per_op["waxpby"].flops + rep.per_op["precond"].flops;
    return {dx.download(), rep};
}

// ---------------------------------------------------------------- byte model (host arithmetic only)
const char* format_name(MatrixFormat f) {
    switch (f) {
        case MatrixFormat::ell: return "ell";
        case MatrixFormat::vt: return "vt";
        case MatrixFormat::pattern: return "pattern";
        default: return "pattern-values";
    }
}
std::optional<MatrixFormat> parse_format(std::string_view name) {
    for (MatrixFormat f : {MatrixFormat::ell, MatrixFormat::vt, MatrixFormat::pattern, MatrixFormat::pattern_with_values})
        if (name == format_name(f)) return f;
    return std::nullopt;
}
const char* limiting_resource_name(LimitingResource r) { return r == LimitingResource::bandwidth ? "bandwidth" : "compute"; }

namespace {
FormatCost finish(ByteBreakdown b, double flops_per_row) {
    FormatCost c;
    c.breakdown = b;
    c.bytes_per_row = b.total();
    c.flops_per_row = flops_per_row;
    c.bytes_per_flop = flops_per_row > 0 ? c.bytes_per_row / flops_per_row : 0.0;
    return c;
}
}  // namespace

FormatCost format_cost(MatrixFormat f, int row_nnz, int table_size, const ModelOptions& opts) {
    ByteBreakdown b;  // inc/perf_model.hpp:49-57: 324 / 116 / 12 / 4 bytes at (27, 2)
    switch (f) {
        case MatrixFormat::ell: b.values = 8.0 * row_nnz; b.indices = 4.0 * row_nnz; break;
        case MatrixFormat::vt: b.indices = 4.0 * row_nnz; b.ends = 4.0 * table_size; break;
        case MatrixFormat::pattern: b.pattern_id = 4.0; b.ends = 4.0 * table_size; break;
        case MatrixFormat::pattern_with_values: b.pattern_id = 4.0; break;
    }
    if (opts.include_input_vector) b.input_vector = 8.0;
    return finish(b, 2.0 * row_nnz);
}
double required_bandwidth(double flops_per_second, const FormatCost& cost) { return flops_per_second * cost.bytes_per_flop; }
RooflineEstimate roofline(const FormatCost& cost, const MachineSpec& machine) {
    RooflineEstimate r;
    r.predicted_flops = machine.read_bandwidth / cost.bytes_per_flop;
    if (machine.peak_flops && *machine.peak_flops < r.predicted_flops) {
        r.predicted_flops = *machine.peak_flops;
        r.limiting_resource = LimitingResource::compute;
    }
    return r;
}
std::vector<ModelRow> model_table(const std::vector<MatrixFormat>& formats, int row_nnz, int table_size, const MachineSpec& machine,
                                  const ModelOptions& opts) {
    std::vector<ModelRow> rows;
    rows.reserve(formats.size());
    for (MatrixFormat f : formats) {
        ModelRow r{f, format_cost(f, row_nnz, table_size, opts), {}};
        r.estimate = roofline(r.cost, machine);
        rows.push_back(r);
    }
    return rows;
}
namespace {
std::string num(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.9g", v);
    return buf;
}
}  // namespace
std::string model_table_csv(const std::vector<ModelRow>& rows) {
    std::string out = "format,bytes_per_row,bytes_per_flop,predicted_gflops,limiting_resource\n";
    for (const ModelRow& r : rows)
        out += std::string(format_name(r.format)) + "," + num(r.cost.bytes_per_row) + "," + num(r.cost.bytes_per_flop) + "," +
               num(r.estimate.predicted_flops / 1e9) + "," + limiting_resource_name(r.estimate.limiting_resource) + "\n";
    return out;
}
std::string model_table_json(const std::vector<ModelRow>& rows) {
    std::string out = "[";
    for (size_t i = 0; i < rows.size(); i++) {
        const ModelRow& r = rows[i];
        out += std::string(i ? ", " : "") + "{\"format\": \"" + format_name(r.format) + "\", \"bytes_per_row\": " + num(r.cost.bytes_per_row) +
               ", \"flops_per_row\": " + num(r.cost.flops_per_row) + ", \"bytes_per_flop\": " + num(r.cost.bytes_per_flop) +
               ", \"predicted_gflops\": " + num(r.estimate.predicted_flops / 1e9) + ", \"limiting_resource\": \"" +
               limiting_resource_name(r.estimate.limiting_resource) + "\"}";
    }
    return out + "]\n";
}
FormatCost measured_cost(const EllMatrix& a) {
    ByteBreakdown b;
    b.values = 8.0 * a.width;
    b.indices = 4.0 * a.width;
    return finish(b, 2.0 * (double)a.nnz / a.n);
}
FormatCost measured_cost(const VtCompressedMatrix& a) {
    ByteBreakdown b;
    b.indices = 4.0 * a.width;
    b.ends = 4.0 * a.table.size();
    return finish(b, 2.0 * (double)a.nnz() / a.n);
}
FormatCost measured_cost(const PatternCompressedMatrix& a) {
    ByteBreakdown b;  // per-row ids, pattern tables amortised; ends per row unless folded (inc/compress.hpp:60-64)
    std::int64_t disp = 0;
    for (const auto& p : a.patterns) disp += (std::int64_t)p.displacements.size();
    b.pattern_id = 4.0;
    b.indices = 4.0 * (double)disp / a.n;
    b.ends = a.values_in_pattern ? 4.0 * a.table.size() * (double)a.patterns.size() / a.n : 4.0 * a.table.size();
    return finish(b, 2.0 * (double)a.nnz() / a.n);
}

}  // namespace spmvcomp

namespace spmvcomp::b200 {
void save_machine_spec(const MachineSpec& machine, const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw IoError("cannot write the machine spec to " + path);
    int ok = std::fprintf(f, "{\"read_bandwidth\": %.17g", machine.read_bandwidth);
    if (ok >= 0 && machine.peak_flops) ok = std::fprintf(f, ", \"peak_flops\": %.17g", *machine.peak_flops);
    if (ok >= 0) ok = std::fprintf(f, "}\n");
    if (std::fclose(f) != 0 || ok < 0) throw IoError("cannot write the machine spec to " + path);
}
MachineSpec load_machine_spec(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "r");
    if (!f) throw IoError("cannot read the machine spec " + path);
    std::string text;
    char buf[256];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) text.append(buf, got);
    std::fclose(f);
    auto field = [&](const char* key) -> std::optional<double> {
        const size_t k = text.find(std::string("\"") + key + "\"");
        if (k == std::string::npos) return std::nullopt;
        const size_t c = text.find(':', k);
        if (c == std::string::npos) return std::nullopt;
        const char* b = text.c_str() + c + 1;
        char* e = nullptr;
        const double v = std::strtod(b, &e);
        if (e == b) return std::nullopt;
        return v;
    };
    MachineSpec m;
    const auto bw = field("read_bandwidth");
    if (!bw || !(*bw > 0.0)) throw IoError("machine spec " + path + ": no positive read_bandwidth");
    m.read_bandwidth = *bw;
    if (const auto pf = field("peak_flops")) {
        if (!(*pf > 0.0)) throw IoError("machine spec " + path + ": peak_flops must be positive");
        m.peak_flops = *pf;
    }
    return m;
}
}  // namespace spmvcomp::b200
