// Vector helpers on the device: make_test_vector (inc/stencil.hpp:54-59) and the
// per-row comparison used by the verification gate.
#include "common.cuh"
#include "hash.cuh"

namespace spmvb {

__global__ void vec_fill_kernel(double *__restrict__ out, int64_t n, int kind, uint64_t seed, double lo, double hi,
                                int64_t first_index) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t g = first_index + i;
        double v;
        if (kind == 0) v = 1.0;
        else if (kind == 1) v = (double)g;
        else {
            // lo + (hi - lo) * u, one rounding per operation (no FMA contraction)
            const double u = u01(h2(seed, (uint64_t)g));
            v = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
        }
        out[i] = v;
    }
}

__global__ void compare_kernel(const double *__restrict__ y, const double *__restrict__ ref,
                               const double *__restrict__ scale, int64_t n, unsigned long long *max_bits,
                               unsigned long long *n_mismatch) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double worst = 0.0;
    unsigned long long bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double a = y[i], b = ref[i];
        if (__double_as_longlong(a) != __double_as_longlong(b)) bad++;
        // with a scale (sum_k |a_ik x_k|, >= |ref|) the deviation is relative to it, which does
        // not blow up on rows whose terms cancel; without one it is relative to |ref|
        double den = scale ? scale[i] : fabs(b);
        if (den == 0.0) den = 1.0;
        double rel = fabs(a - b) / den;
        if (!(rel == rel)) rel = INFINITY;  // NaN anywhere is a failure
        worst = fmax(worst, rel);
    }
    for (int o = 16; o > 0; o >>= 1) {
        worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(max_bits, (unsigned long long)__double_as_longlong(worst));  // worst >= 0: order preserving
        if (bad) atomicAdd(n_mismatch, bad);
    }
}

__global__ void row_abs_scale_kernel(const int64_t *__restrict__ row_start, const int32_t *__restrict__ cols,
                                     const double *__restrict__ vals, const double *__restrict__ x, int64_t x_col0,
                                     double *__restrict__ scale, int n) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double acc = 0.0;
    for (int64_t t = row_start[r]; t < row_start[r + 1]; t++)
        acc = __dadd_rn(acc, fabs(__dmul_rn(vals[t], x[(int64_t)cols[t] - x_col0])));
    scale[r] = acc;
}

}  // namespace spmvb

using namespace spmvb;

extern "C" {

int spmvb_vec_fill(double *dev, int64_t n, int32_t kind, uint64_t seed, double lo, double hi, int64_t first_index,
                   void *stream) {
    if (!dev || n < 0 || kind < 0 || kind > 2) return fail(SPMVB_ERR_INVALID_ARGUMENT, "vec_fill: bad arguments");
    if (n == 0) return SPMVB_OK;
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((n + threads - 1) / threads, sm_count() * 16);
    vec_fill_kernel<<<blocks, threads, 0, as_stream(stream)>>>(dev, n, kind, seed, lo, hi, first_index);
    SPMVB_CUDA(cudaGetLastError());
    return SPMVB_OK;
}

int spmvb_compare(const double *y, const double *ref, const double *scale, int64_t n, double *max_rel,
                  int64_t *n_bit_mismatch, void *stream) {
    if (!y || !ref || n < 0) return fail(SPMVB_ERR_INVALID_ARGUMENT, "compare: bad arguments");
    unsigned long long *d = nullptr;
    SPMVB_CUDA(cudaMalloc(&d, 16));
    SPMVB_CUDA(cudaMemsetAsync(d, 0, 16, as_stream(stream)));
    if (n > 0) {
        const int threads = 256;
        const int blocks = (int)std::min<int64_t>((n + threads - 1) / threads, sm_count() * 16);
        compare_kernel<<<blocks, threads, 0, as_stream(stream)>>>(y, ref, scale, n, d, d + 1);
    }
    unsigned long long h[2] = {0, 0};
    cudaError_t e = cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, as_stream(stream));
    if (e == cudaSuccess) e = cudaStreamSynchronize(as_stream(stream));
    cudaFree(d);
    if (e != cudaSuccess) return fail(SPMVB_ERR_CUDA, "compare failed: %s", cudaGetErrorString(e));
    if (max_rel) memcpy(max_rel, &h[0], 8);
    if (n_bit_mismatch) *n_bit_mismatch = (int64_t)h[1];
    return SPMVB_OK;
}

int spmvb_row_abs_scale(const spmvb_matrix *csr, const double *x_dev, int64_t x_col0, double *scale_dev,
                        void *stream) {
    if (!csr || csr->format != SPMVB_FMT_CSR || !x_dev || !scale_dev)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "row_abs_scale: needs a CSR handle");
    if (csr->n == 0) return SPMVB_OK;
    row_abs_scale_kernel<<<(csr->n + 255) / 256, 256, 0, as_stream(stream)>>>(
        static_cast<const int64_t *>(csr->s[SPMVB_S_CSR_ROW_START]), static_cast<const int32_t *>(csr->s[SPMVB_S_CSR_COLS]),
        static_cast<const double *>(csr->s[SPMVB_S_CSR_VALS]), x_dev, x_col0, scale_dev, csr->n);
    SPMVB_CUDA(cudaGetLastError());
    return SPMVB_OK;
}

}  // extern "C"
