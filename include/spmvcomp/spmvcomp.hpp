// spmvcomp.hpp -- the `spmvcomp` C++ API for the SpMV path, as implemented by the
// B200-native library.  Names, fields, signatures and error behaviour are those of
// the reference's public headers (cited per declaration as inc/<file>:<line> under
// /root/reference/proj/include/spmvcomp), so code written against the reference
// compiles against this header unchanged; the per-topic headers next to this file
// (grid.hpp, stencil.hpp, ...) forward here.  Every function below runs on the GPU
// through the C-ABI in spmvcomp_b200.h -- there is no CPU implementation.
//
// Declared here: everything on the SpMV path and its first
// caller, the CG driver with dot / waxpby / symgs_sweep (section 8f rows N1, N4).
// Not declared: the model_table* emitters (tooling outside the path).  File formats: spmvcomp/io.hpp.
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <filesystem>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace spmvcomp {

// ---------------------------------------------------------------- errors (inc/errors.hpp:9-42)
struct TableOverflowError : std::runtime_error {  // more distinct values than the table limit
    explicit TableOverflowError(const std::string& m) : std::runtime_error(m) {}
};
struct IntegrityError : std::runtime_error {  // a compressed structure violates its invariants
    explicit IntegrityError(const std::string& m) : std::runtime_error(m) {}
};
struct VerificationError : std::runtime_error {  // a kernel's output did not match the ELL baseline
    explicit VerificationError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
class DivergenceError : public std::runtime_error {
public:
    DivergenceError(int iteration, const std::string& m) : std::runtime_error(m), it_(iteration) {}
    int iteration() const noexcept { return it_; }

private:
    int it_;
};

// ---------------------------------------------------------------- geometry (inc/grid.hpp:11-47)
inline constexpr std::int64_t kMaxRows = (std::int64_t{1} << 31) - 1;  // columns are 4-byte signed

struct GridSpec {  // x-fastest numbering: row = ix + nx*(iy + ny*iz)
    int nx = 1, ny = 1, nz = 1;
    std::int64_t rows() const { return std::int64_t{nx} * ny * nz; }
    bool known() const { return nx > 0 && ny > 0 && nz > 0; }
    std::int64_t node(int ix, int iy, int iz) const { return ix + std::int64_t{nx} * (iy + std::int64_t{ny} * iz); }
    friend bool operator==(const GridSpec&, const GridSpec&) = default;
};

inline void validate(const GridSpec& g) {
    const std::string dims = std::to_string(g.nx) + "x" + std::to_string(g.ny) + "x" + std::to_string(g.nz);
    if (g.nx < 1 || g.ny < 1 || g.nz < 1) throw std::invalid_argument("grid dimensions must be >= 1, got " + dims);
    if (g.rows() > kMaxRows)
        throw std::invalid_argument("grid " + dims + " has " + std::to_string(g.rows()) +
                                    " rows; column indices must fit a 4-byte signed integer");
}

// ---------------------------------------------------------------- matrices and vectors
using Vector = std::vector<double>;  // inc/stencil.hpp:14

struct StencilMatrix {  // CSR, columns strictly ascending per row (inc/stencil.hpp:19-36)
    std::int32_t n = 0;
    std::vector<std::int64_t> row_start;  // n + 1
    std::vector<std::int32_t> cols;
    std::vector<double> vals;
    GridSpec grid{0, 0, 0};  // provenance; not part of equality

    std::int64_t nnz() const { return row_start.empty() ? 0 : row_start[n]; }
    std::int32_t row_nnz(std::int32_t i) const { return static_cast<std::int32_t>(row_start[i + 1] - row_start[i]); }
    std::span<const std::int32_t> row_cols(std::int32_t i) const {
        return {cols.data() + row_start[i], static_cast<std::size_t>(row_nnz(i))};
    }
    std::span<const double> row_vals(std::int32_t i) const {
        return {vals.data() + row_start[i], static_cast<std::size_t>(row_nnz(i))};
    }
};
bool operator==(const StencilMatrix& a, const StencilMatrix& b);  // inc/stencil.hpp:38

// inc/stencil.hpp:40-45: 27-point stencil, out-of-grid couplings omitted, HPCG values by default
StencilMatrix generate_matrix(const GridSpec& spec, double diagonal = 26.0, double off_diagonal = -1.0);
// inc/stencil.hpp:47-50: explicit rows; columns strictly ascending and in [0, n)
StencilMatrix stencil_from_rows(std::int32_t n, const std::vector<std::vector<std::pair<std::int32_t, double>>>& rows);
bool is_symmetric(const StencilMatrix& m);  // inc/stencil.hpp:52

// inc/stencil.hpp:61-64: coordinate format, 1-based, lower triangle only; the matrix must be symmetric (spmvcomp/io.hpp)
void write_matrix_market(const StencilMatrix& m, const std::filesystem::path& path);

enum class VectorKind { ones, linear, random };  // inc/stencil.hpp:54
// inc/stencil.hpp:56-59: random is deterministic in [0,1) per seed; the seed is required for it
Vector make_test_vector(std::int64_t n, VectorKind kind, std::optional<std::uint64_t> seed = std::nullopt);

struct EllMatrix {  // row-major padded ELL; padding = (0.0, own row) (inc/ell.hpp:10-24)
    std::int32_t n = 0, width = 0;
    std::int64_t nnz = 0;
    std::vector<double> values;         // n * width
    std::vector<std::int32_t> columns;  // n * width
    std::int64_t slot(std::int32_t row, std::int32_t k) const { return std::int64_t{row} * width + k; }
};
bool operator==(const EllMatrix& a, const EllMatrix& b);
EllMatrix to_ell(const StencilMatrix& m);      // inc/ell.hpp:28-29
StencilMatrix to_stencil(const EllMatrix& a);  // inc/ell.hpp:31-32

struct ValueTable {  // strictly ascending distinct values, bit-pattern equality (inc/compress.hpp:11-20)
    std::vector<double> entries;
    std::int32_t size() const { return static_cast<std::int32_t>(entries.size()); }
    double operator[](std::int32_t k) const { return entries[k]; }
    friend bool operator==(const ValueTable&, const ValueTable&) = default;
};
struct CompressOptions {  // inc/compress.hpp:22-26
    std::size_t value_table_limit = 256;
};

struct VtCompressedMatrix {  // inc/compress.hpp:28-44
    std::int32_t n = 0, width = 0;
    ValueTable table;
    std::vector<std::int32_t> sorted_columns;  // n * width, (value, column) order, padding = own row
    std::vector<std::int32_t> ends;            // n * table.size(), exclusive group ends
    std::int64_t nnz() const;
    std::int32_t row_nnz(std::int32_t i) const { return ends[(i + 1) * std::int64_t{table.size()} - 1]; }
};
bool operator==(const VtCompressedMatrix& a, const VtCompressedMatrix& b);

struct DisplacementPattern {  // inc/compress.hpp:48-58
    std::vector<std::int32_t> displacements;  // column - row, (value, displacement) order
    std::vector<std::int32_t> ends;           // table.size() exclusive group ends
    friend bool operator==(const DisplacementPattern&, const DisplacementPattern&) = default;
    friend auto operator<=>(const DisplacementPattern&, const DisplacementPattern&) = default;
};
struct PatternCompressedMatrix {  // inc/compress.hpp:60-76
    std::int32_t n = 0;
    ValueTable table;
    std::vector<DisplacementPattern> patterns;
    std::vector<std::int32_t> row_pattern;  // n ids
    bool values_in_pattern = false;
    std::int64_t nnz() const;
    std::int32_t row_nnz(std::int32_t i) const { return patterns[row_pattern[i]].ends.back(); }
};
bool operator==(const PatternCompressedMatrix& a, const PatternCompressedMatrix& b);

ValueTable scan_value_table(const StencilMatrix& m, std::size_t limit);                           // inc/compress.hpp:80
VtCompressedMatrix compress_values(const StencilMatrix& m, const CompressOptions& opts = {});     // inc/compress.hpp:82
PatternCompressedMatrix compress_patterns(const StencilMatrix& m, bool values_in_pattern,         // inc/compress.hpp:84-85
                                          const CompressOptions& opts = {});
StencilMatrix decompress(const VtCompressedMatrix& c);       // inc/compress.hpp:87-90
StencilMatrix decompress(const PatternCompressedMatrix& c);
void validate(const VtCompressedMatrix& c);                  // inc/compress.hpp:92-95, IntegrityError
void validate(const PatternCompressedMatrix& c);

// ---------------------------------------------------------------- kernels (inc/kernels.hpp:12-37)
inline std::int64_t spmv_flops(std::int64_t nnz) { return 2 * nnz; }
inline std::int64_t dot_flops(std::int64_t n) { return 2 * n; }
inline std::int64_t waxpby_flops(std::int64_t n) { return 2 * n; }
inline std::int64_t symgs_flops(std::int64_t nnz) { return 4 * nnz; }

// y = A x, overwrite; inputs validated (length mismatch -> std::invalid_argument).
Vector spmv(const EllMatrix& a, const Vector& x);
Vector spmv(const VtCompressedMatrix& a, const Vector& x);
Vector spmv(const PatternCompressedMatrix& a, const Vector& x);

namespace unchecked {  // rows [begin, end) of pre-validated inputs; other rows of y untouched
void spmv_rows(const EllMatrix& a, std::span<const double> x, std::span<double> y, std::int32_t begin, std::int32_t end);
void spmv_rows(const VtCompressedMatrix& a, std::span<const double> x, std::span<double> y, std::int32_t begin,
               std::int32_t end);
void spmv_rows(const PatternCompressedMatrix& a, std::span<const double> x, std::span<double> y, std::int32_t begin,
               std::int32_t end);
}  // namespace unchecked

// ---------------------------------------------------------------- CG caller (inc/kernels.hpp:39-42, inc/solver.hpp:13-46)
double dot(const Vector& u, const Vector& v);                                               // length mismatch -> invalid_argument
Vector waxpby(double alpha, const Vector& x, double beta, const Vector& y);                 // w = alpha*x + beta*y
void waxpby_into(double alpha, const Vector& x, double beta, const Vector& y, Vector& w);
// inc/kernels.hpp:44-48: forward then backward Gauss-Seidel sweep in natural order, in place.  On the device the rows run by
// hyperplanes of the matrix's grid (m.grid; results bit-identical to the sequential loop); std::invalid_argument for a zero
// diagonal, a length mismatch, or a matrix without grid provenance / with couplings outside the 27-point neighbourhood.
void symgs_sweep(const StencilMatrix& m, Vector& x, const Vector& b);

enum class SpmvBackend { ell, vt, pattern };
const char* backend_name(SpmvBackend b);

struct CgConfig {
    int max_iterations = 500;
    double tolerance = 1e-8;  // relative residual ||r||2 / ||b||2
    int symgs_sweeps = 0;     // 0 = unpreconditioned; >= 1: SymGS sweeps from a zero guess (needs m.grid, see symgs_sweep)
    SpmvBackend backend = SpmvBackend::ell;
};
struct OpStats {
    std::int64_t calls = 0, flops = 0;
    double seconds = 0.0;
};
struct CgReport {
    int iterations = 0;
    bool converged = false;
    std::vector<double> residual_history;  // iterations + 1 entries, [0] = 1.0
    std::int64_t flops_total = 0;
    std::map<std::string, OpStats> per_op;  // "spmv", "dot", "waxpby", "precond"
    double final_residual() const { return residual_history.back(); }
};
// x0 = 0; per iteration exactly 1 SpMV (on the configured backend), 3 dots and 3 waxpbys, all on the GPU.
std::pair<Vector, CgReport> cg_solve(const StencilMatrix& m, const Vector& b, const CgConfig& cfg = {});

// ---------------------------------------------------------------- byte model (inc/perf_model.hpp:14-80)
enum class MatrixFormat { ell, vt, pattern, pattern_with_values };
const char* format_name(MatrixFormat f);
std::optional<MatrixFormat> parse_format(std::string_view name);

struct MachineSpec {
    double read_bandwidth = 75e9;
    std::optional<double> peak_flops;
};
struct ByteBreakdown {
    double values = 0, indices = 0, ends = 0, pattern_id = 0, input_vector = 0;
    double total() const { return values + indices + ends + pattern_id + input_vector; }
    friend bool operator==(const ByteBreakdown&, const ByteBreakdown&) = default;
};
struct FormatCost {
    double bytes_per_row = 0, flops_per_row = 0, bytes_per_flop = 0;
    ByteBreakdown breakdown;
};
struct ModelOptions {
    bool include_input_vector = false;
};
FormatCost format_cost(MatrixFormat f, int row_nnz, int table_size, const ModelOptions& opts = {});
double required_bandwidth(double flops_per_second, const FormatCost& cost);
enum class LimitingResource { bandwidth, compute };
const char* limiting_resource_name(LimitingResource r);
struct RooflineEstimate {
    double predicted_flops = 0;
    LimitingResource limiting_resource = LimitingResource::bandwidth;
};
RooflineEstimate roofline(const FormatCost& cost, const MachineSpec& machine);
FormatCost measured_cost(const EllMatrix& a);
FormatCost measured_cost(const VtCompressedMatrix& a);
FormatCost measured_cost(const PatternCompressedMatrix& a);

// inc/perf_model.hpp:82-95: one row per format -- cost of a row with row_nnz entries and the roofline estimate on `machine`
struct ModelRow {
    MatrixFormat format;
    FormatCost cost;
    RooflineEstimate estimate;
};
std::vector<ModelRow> model_table(const std::vector<MatrixFormat>& formats, int row_nnz, int table_size, const MachineSpec& machine,
                                  const ModelOptions& opts = {});
// CSV columns, in order: format, bytes_per_row, bytes_per_flop, predicted_gflops, limiting_resource
std::string model_table_csv(const std::vector<ModelRow>& rows);
std::string model_table_json(const std::vector<ModelRow>& rows);

}  // namespace spmvcomp
