// CG vector primitives and the unpreconditioned CG driver on the device
// (inc/kernels.hpp:39-42 dot / waxpby, inc/solver.hpp:17-46 CgConfig / CgReport / cg_solve;
// SPEC.md:238-256,308-321).  The caller of the SpMV hot path: 1 SpMV, 3 dots and 3 waxpbys
// per iteration (inc/solver.hpp:43), everything device-resident; only the three dot results
// per iteration cross to the host (they steer alpha, beta and the stopping test).
//
// waxpby is bit-identical to the reference expression alpha*x[i] + beta*y[i] (two products and
// one sum, each rounded).  dot uses a fixed-shape two-level tree (deterministic run to run) and
// therefore differs from the reference's index-ascending sum in the last bits
// bounds that effect on the residual history by 1e-10.
#include <cmath>
#include <vector>

#include "common.cuh"

namespace spmvb {

constexpr int kDotBlocks = 148 * 4;
constexpr int kDotThreads = 256;

__global__ void __launch_bounds__(kDotThreads) dot_partial_kernel(const double *__restrict__ u, const double *__restrict__ v,
                                                                 int64_t n, double *__restrict__ partial) {
    // each thread: ascending strided sum; block: fixed shuffle / shared-memory tree
    __shared__ double s[kDotThreads / 32];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kDotThreads)
        acc = __dadd_rn(acc, __dmul_rn(u[i], v[i]));
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < kDotThreads / 32 ? s[threadIdx.x] : 0.0;
        for (int o = 4; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
        if (threadIdx.x == 0) partial[blockIdx.x] = acc;
    }
}

__global__ void dot_final_kernel(const double *__restrict__ partial, int count, double *__restrict__ out) {
    // one warp, ascending chunks then a fixed tree: order independent of scheduling
    double acc = 0.0;
    for (int i = threadIdx.x; i < count; i += 32) acc = __dadd_rn(acc, partial[i]);
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
    if (threadIdx.x == 0) *out = acc;
}

__global__ void waxpby_kernel(double alpha, const double *__restrict__ x, double beta, const double *__restrict__ y,
                              double *__restrict__ w, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        w[i] = __dadd_rn(__dmul_rn(alpha, x[i]), __dmul_rn(beta, y[i]));  // inc/kernels.hpp:41
}

struct DotScratch {
    double *partial = nullptr, *out = nullptr;
    ~DotScratch() {
        if (partial) cudaFree(partial);
        if (out) cudaFree(out);
    }
    int init() {
        SPMVB_CUDA(cudaMalloc(&partial, kDotBlocks * sizeof(double)));
        SPMVB_CUDA(cudaMalloc(&out, sizeof(double)));
        return SPMVB_OK;
    }
};

static int dot_device(const double *u, const double *v, int64_t n, DotScratch &sc, double *host, cudaStream_t st) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + kDotThreads - 1) / kDotThreads, kDotBlocks));
    dot_partial_kernel<<<blocks, kDotThreads, 0, st>>>(u, v, n, sc.partial);
    dot_final_kernel<<<1, 32, 0, st>>>(sc.partial, blocks, sc.out);
    SPMVB_CUDA(cudaMemcpyAsync(host, sc.out, sizeof(double), cudaMemcpyDeviceToHost, st));
    SPMVB_CUDA(cudaStreamSynchronize(st));
    return SPMVB_OK;
}

static int waxpby_device(double alpha, const double *x, double beta, const double *y, double *w, int64_t n, cudaStream_t st) {
    if (n <= 0) return SPMVB_OK;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    waxpby_kernel<<<blocks, 256, 0, st>>>(alpha, x, beta, y, w, n);
    SPMVB_CUDA(cudaGetLastError());
    return SPMVB_OK;
}

}  // namespace spmvb

using namespace spmvb;

extern "C" {

int spmvb_dot(const double *u_dev, const double *v_dev, int64_t n, double *result, void *stream) {
    if (!u_dev || !v_dev || !result || n < 0) return fail(SPMVB_ERR_INVALID_ARGUMENT, "dot: bad arguments");
    DotScratch sc;
    SPMVB_TRY(sc.init());
    return dot_device(u_dev, v_dev, n, sc, result, as_stream(stream));
}

int spmvb_waxpby(double alpha, const double *x_dev, double beta, const double *y_dev, double *w_dev, int64_t n, void *stream) {
    if (!x_dev || !y_dev || !w_dev || n < 0) return fail(SPMVB_ERR_INVALID_ARGUMENT, "waxpby: bad arguments");
    return waxpby_device(alpha, x_dev, beta, y_dev, w_dev, n, as_stream(stream));
}

int spmvb_cg_solve(const spmvb_matrix *a, const double *b_dev, double *x_dev, int32_t max_iterations, double tolerance,
                   int32_t *iterations, int32_t *converged, double *residual_history, void *stream) {
    if (!a || !b_dev || !x_dev || !iterations || !converged)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "cg_solve: NULL argument");
    if (max_iterations < 1 || !(tolerance > 0.0))
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "cg_solve: need max_iterations >= 1 and tolerance > 0");
    if (a->row_offset != 0) return fail(SPMVB_ERR_INVALID_ARGUMENT, "cg_solve: handle is a slab; drive the slabs from slab.py");
    cudaStream_t st = as_stream(stream);
    const int64_t n = a->n;
    *iterations = 0;
    *converged = 0;
    double *r = nullptr, *p = nullptr, *ap = nullptr;
    DotScratch sc;
    SPMVB_TRY(sc.init());
    int rc = spmvb_vec_alloc(n, &r);
    if (rc == SPMVB_OK) rc = spmvb_vec_alloc(n, &p);
    if (rc == SPMVB_OK) rc = spmvb_vec_alloc(n, &ap);
    auto done = [&](int code) {
        if (r) cudaFree(r);
        if (p) cudaFree(p);
        if (ap) cudaFree(ap);
        return code;
    };
    if (rc != SPMVB_OK) return done(rc);
    // x0 = 0, r = b, z = r (no preconditioner), p = z  (inc/solver.hpp:40-43)
    rc = cudaMemsetAsync(x_dev, 0, (size_t)n * 8, st) == cudaSuccess ? SPMVB_OK : fail(SPMVB_ERR_CUDA, "memset failed");
    if (rc == SPMVB_OK) rc = waxpby_device(1.0, b_dev, 0.0, b_dev, r, n, st);
    if (rc == SPMVB_OK) rc = waxpby_device(1.0, r, 0.0, r, p, n, st);
    double bb = 0.0, rz = 0.0;
    if (rc == SPMVB_OK) rc = dot_device(b_dev, b_dev, n, sc, &bb, st);
    if (rc != SPMVB_OK) return done(rc);
    const double bnorm = std::sqrt(bb);
    rz = bb;
    if (residual_history) residual_history[0] = 1.0;
    if (bnorm == 0.0) {  // b = 0: x = 0 is the solution
        *converged = 1;
        return done(SPMVB_OK);
    }
    for (int it = 1; it <= max_iterations; it++) {
        double pap = 0.0, rr = 0.0, rz_new = 0.0;
        rc = spmvb_spmv(a, p, 0, n, ap, 0, (int32_t)n, stream);                       // 1 SpMV
        if (rc == SPMVB_OK) rc = dot_device(p, ap, n, sc, &pap, st);                   // dot 1
        if (rc != SPMVB_OK) return done(rc);
        const double alpha = rz / pap;
        rc = waxpby_device(1.0, x_dev, alpha, p, x_dev, n, st);                        // waxpby 1
        if (rc == SPMVB_OK) rc = waxpby_device(1.0, r, -alpha, ap, r, n, st);          // waxpby 2
        if (rc == SPMVB_OK) rc = dot_device(r, r, n, sc, &rr, st);                     // dot 2 (residual norm)
        if (rc == SPMVB_OK) rc = dot_device(r, r, n, sc, &rz_new, st);                 // dot 3 (r.z with z = r)
        if (rc != SPMVB_OK) return done(rc);
        const double rel = std::sqrt(rr) / bnorm;
        *iterations = it;
        if (residual_history) residual_history[it] = rel;
        if (!std::isfinite(alpha) || !std::isfinite(rel)) {
            done(SPMVB_OK);
            return fail(SPMVB_ERR_DIVERGENCE, "cg_solve: non-finite value in iteration %d", it);  // inc/solver.hpp:44
        }
        if (rel <= tolerance) {
            *converged = 1;
            break;
        }
        const double beta = rz_new / rz;
        rz = rz_new;
        rc = waxpby_device(1.0, r, beta, p, p, n, st);                                 // waxpby 3: p = z + beta p
        if (rc != SPMVB_OK) return done(rc);
    }
    SPMVB_CUDA(cudaStreamSynchronize(st));
    return done(SPMVB_OK);
}

}  // extern "C"
