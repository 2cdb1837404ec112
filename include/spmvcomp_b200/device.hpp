// device.hpp -- B200 extension of the spmvcomp C++ API: device-resident matrices and
// vectors for callers that run many SpMVs (the benchmark loop, CG), so that only the
// first call pays the upload.  Thin RAII wrappers over the C-ABI (spmvcomp_b200.h).
#pragma once

#include <cstdint>
#include <span>
#include <string>

#include "spmvcomp/compress.hpp"
#include "spmvcomp/ell.hpp"
#include "spmvcomp/errors.hpp"
#include "spmvcomp/grid.hpp"
#include "spmvcomp/kernels.hpp"
#include "spmvcomp/stencil.hpp"
#include "spmvcomp_b200.h"

namespace spmvcomp::b200 {

// Throws the reference exception that corresponds to a C-ABI status (inc/errors.hpp).
void throw_on_error(int status);

struct HybridOptions {          // exception-row extension
    std::int32_t min_pattern_rows = 2;
    std::int32_t dict_cap = 0;
};

class DeviceMatrix {
public:
    DeviceMatrix() = default;
    explicit DeviceMatrix(spmvb_matrix* h) : h_(h) {}
    explicit DeviceMatrix(const StencilMatrix& m);
    explicit DeviceMatrix(const EllMatrix& a);
    explicit DeviceMatrix(const VtCompressedMatrix& a);
    explicit DeviceMatrix(const PatternCompressedMatrix& a);
    DeviceMatrix(DeviceMatrix&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    DeviceMatrix& operator=(DeviceMatrix&& o) noexcept;
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
    ~DeviceMatrix();

    spmvb_matrix* handle() const { return h_; }
    spmvb_matrix_info info() const;

    // device-side build (generate_matrix / to_ell / compress_* without a host round trip)
    static DeviceMatrix generate(const GridSpec& spec, double diagonal = 26.0, double off_diagonal = -1.0,
                                 std::int64_t row_begin = 0, std::int64_t row_end = -1);
    DeviceMatrix to_ell(std::int32_t min_width = 0) const;
    DeviceMatrix compress_values(const CompressOptions& o = {}, std::int32_t min_width = 0) const;
    DeviceMatrix compress_patterns(bool values_in_pattern, const CompressOptions& o = {}) const;
    DeviceMatrix compress_hybrid(bool values_in_pattern, const HybridOptions& h = {}, const CompressOptions& o = {}) const;
    DeviceMatrix to_csr() const;

    StencilMatrix download_csr() const;
    EllMatrix download_ell() const;
    VtCompressedMatrix download_vt() const;
    PatternCompressedMatrix download_pattern() const;  // throws if the handle holds exception rows

private:
    spmvb_matrix* h_ = nullptr;
};

class DeviceVector {
public:
    explicit DeviceVector(std::int64_t n);
    explicit DeviceVector(std::span<const double> host);
    DeviceVector(DeviceVector&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
    DeviceVector(const DeviceVector&) = delete;
    DeviceVector& operator=(const DeviceVector&) = delete;
    ~DeviceVector();
    double* data() const { return p_; }
    std::int64_t size() const { return n_; }
    void upload(std::span<const double> host);
    Vector download() const;
    void fill(VectorKind kind, std::uint64_t seed = 0, double lo = 0.0, double hi = 1.0, std::int64_t first_index = 0);

private:
    double* p_ = nullptr;
    std::int64_t n_ = 0;
};

// unchecked::spmv_rows on device-resident data, asynchronous on `stream` (a cudaStream_t).
void spmv_rows(const DeviceMatrix& a, const DeviceVector& x, DeviceVector& y, std::int32_t begin, std::int32_t end,
               void* stream = nullptr);

// The machine-spec file `calibrate` writes and `bench --machine` reads (the reference names no layout: one JSON
// object {"read_bandwidth": bytes/s[, "peak_flops": flops/s]}, numbers with 17 significant digits so that a round trip is exact).
// IoError for unreadable / unwritable files and for text without a positive read_bandwidth.
void save_machine_spec(const MachineSpec& machine, const std::string& path);
MachineSpec load_machine_spec(const std::string& path);

}  // namespace spmvcomp::b200
