// Host-side entry points shared between the SpMV translation units.
#pragma once
#include "common.cuh"

namespace spmvb {

struct PatternArgs;

int check_launch(const char *what);
// ELL rows [row_begin,row_end); row_map != nullptr serves the exception block (rows = exception slots)
int launch_ell(const double *values, const int32_t *columns, int width, const double *x, int64_t x_col0, double *y,
               int row_begin, int row_end, const int32_t *row_map, cudaStream_t st);
// exception rows [e_begin,e_end) of a hybrid pattern handle from shared-memory windows of x (spmv_exception.cu):
// 0 launched, 1 not served (run launch_ell with the row map), < 0 error
int launch_exception_window(const spmvb_matrix *a, const double *x, int64_t x_col0, int64_t x_len, double *y, int e_begin, int e_end,
                            cudaStream_t st);
int launch_vt(const spmvb_matrix *a, const double *x, int64_t x_col0, double *y, int row_begin, int row_end, cudaStream_t st);
// measured experiments (spmv_pattern_lab.cu): returns 0 launched, 1 not served, -1 CUDA error
int launch_pattern_lab(int which, const spmvb_matrix *a, PatternArgs &p, cudaStream_t st);

// Request of cg_solve to the next spmvb_spmv of this host thread: also leave partial sums of x.y (y = A x, square full-grid
// handle).  Served only by the default tensor-ring launch (count = partials written, one per warp); count stays 0 when the
// launch that ran could not serve it, and the caller then runs its own dot.  The partials are summed in a fixed order
// (each thread over its rows in schedule order, a shuffle tree per warp), so the result is deterministic run to run.
struct FusedDot {
    double *partial = nullptr;
    int capacity = 0, count = 0;
};
FusedDot *&fused_dot_request();

// tensor-ring kernel (spmv_pattern_tma.cu): same return convention; `which` selects a measured variant
bool ring_ok(const spmvb_matrix *a, const PatternArgs &p);
int launch_pattern_ring(int which, int lines, const spmvb_matrix *a, PatternArgs &p, cudaStream_t st);

}  // namespace spmvb
