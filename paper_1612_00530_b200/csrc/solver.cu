// CG vector primitives and the unpreconditioned CG driver on the device
// (inc/kernels.hpp:39-42 dot / waxpby, inc/solver.hpp:17-46 CgConfig / CgReport / cg_solve;
// SPEC.md:238-256,308-321).  The caller of the SpMV hot path: 1 SpMV, 3 dots and 3 waxpbys
// per iteration (inc/solver.hpp:43), everything device-resident.  Inside cg_solve the operations of an
// iteration are fused where that saves passes over the vectors -- x and r are updated and r.r is
// accumulated in one kernel, alpha and beta are formed on the device -- with exactly the arithmetic
// and summation order of the stand-alone dot / waxpby; one pair of scalars (alpha, r.r) per iteration
// crosses to the host for the history and the stopping test.
//
// waxpby is bit-identical to the reference expression alpha*x[i] + beta*y[i] (two products and
// one sum, each rounded).  dot uses a fixed-shape two-level tree (deterministic run to run) and
// therefore differs from the reference's index-ascending sum in the last bits
// bounds that effect on the residual history by 1e-10.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "device_utils.cuh"
#include "spmv_internal.cuh"

namespace spmvb {

// Shape of the reduction tree of dot (part of the result's bits, so a constant, not the device's SM count): 1184 partial sums.
constexpr int kDotBlocks = 1184;
constexpr int kDotThreads = 256;
constexpr int kPartialCap = 8192;  // partial sums: kDotBlocks from the vector kernels, one per warp from the SpMV's fused dot

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

// Sum of `count` partial sums in the fixed order of dot_final_kernel (lane l: partial[l], partial[l+32], ... ascending, then the
// shuffle tree), by the first warp of a block whose threads ALL fetch: the values land in shared memory in one round of
// loads (ld.global.cg: written by other blocks / the previous kernel), then lane l adds its own in order.  A lane-serial loop of
// dependent global loads took 7 us for 1184 values (the round-1 alpha / beta kernels).  Result valid in thread 0.
constexpr int kSumChunk = 2048;
__device__ __forceinline__ double block_ordered_sum(const double *partial, int count, double *buf /* kSumChunk doubles, shared */) {
    double acc = 0.0;
    for (int base = 0; base < count; base += kSumChunk) {
        const int m = min(kSumChunk, count - base);
        for (int i = threadIdx.x; i < m; i += blockDim.x) buf[i] = __ldcg(partial + base + i);
        __syncthreads();
        if (threadIdx.x < 32)
            for (int i = threadIdx.x; i < m; i += 32) acc = __dadd_rn(acc, buf[i]);
        __syncthreads();
    }
    if (threadIdx.x < 32)
        for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
    return acc;
}

__global__ void dot_final_kernel(const double *__restrict__ partial, int count, double *__restrict__ out) {
    // one warp's order -- ascending lane-strided sums, then a fixed tree: independent of scheduling -- fetched by the whole block
    __shared__ double s_buf[kSumChunk];
    const double acc = block_ordered_sum(partial, count, s_buf);
    if (threadIdx.x == 0) *out = acc;
}

__global__ void waxpby_kernel(double alpha, const double *__restrict__ x, double beta, const double *__restrict__ y,
                              double *__restrict__ w, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        w[i] = __dadd_rn(__dmul_rn(alpha, x[i]), __dmul_rn(beta, y[i]));  // inc/kernels.hpp:41
}

// ---- fused forms used by cg_solve (same per-element expressions, same reduction tree as dot_partial_kernel) ----
// scal: [0] p.Ap  [1] alpha  [2] r.z of the previous iteration  [3] r.r (= r.z, no preconditioner)  [4] beta
//       [5] stop flag (set by the device when the iteration converged or produced a non-finite value; every later
//           cg_* kernel is then a no-op, so the host may queue one iteration ahead)  [6] ||b||  [7] tolerance  [8] ||r||/||b||
__global__ void cg_alpha_kernel(const double *__restrict__ partial, int count, double *__restrict__ scal) {
    if (scal[5] != 0.0) return;
    __shared__ double s_buf[kSumChunk];
    const double acc = block_ordered_sum(partial, count, s_buf);
    if (threadIdx.x == 0) {
        scal[0] = acc;
        scal[1] = scal[2] / acc;  // alpha = r.z / p.Ap
    }
}
// The iteration's vector kernel ("cg_fused_scalars"): the two updates, r.r, and -- by the block that finishes last (a ticket
// counter) -- what cg_beta_kernel did: the partial sums of r.r added in that kernel's order, beta, stop flag, iteration count, the
// record into the host's pinned ring.  alpha comes from cg_alpha_kernel (pap_partial == NULL) or, variant 2, is formed at the head
// by every block from the partial sums of p.Ap (cg_alpha_kernel's order: the same bits in every block).  At most 32 registers:
// 1184 blocks of 256 threads are exactly one wave, and one register more makes that two (measured: 119 -> 164 us at 256^3).
__global__ void __launch_bounds__(kDotThreads, 8) cg_update_fused_kernel(double *__restrict__ scal, const double *__restrict__ p,
                                                                     const double *__restrict__ ap, double *__restrict__ x,
                                                                     double *__restrict__ r, int64_t n, const double *pap_partial, int pap_count,
                                                                     double *partial, unsigned int *ticket, double *host_ring, int ring_slots) {
    __shared__ double s[kDotThreads / 32];
    __shared__ double s_alpha;
    __shared__ int s_last;
    __shared__ double s_buf[kSumChunk];
    pdl_launch_dependents();
    pdl_grid_dependency_wait();
    if (scal[5] != 0.0) return;
    // alpha: from cg_alpha_kernel (pap_partial == NULL), or formed here by every block from the partial sums of p.Ap (measured
    // slower: 1184 blocks reading the same 74 lines of L2 at once cost 45 us at 256^3 -- kept for the record, not used)
    double pap_sum = 0.0;  // thread 0: p.Ap
    if (pap_partial) {
        pap_sum = block_ordered_sum(pap_partial, pap_count, s_buf);
        if (threadIdx.x == 0) s_alpha = scal[2] / pap_sum;  // alpha = r.z / p.Ap
    } else if (threadIdx.x == 0) {
        pap_sum = scal[0];
        s_alpha = scal[1];
    }
    __syncthreads();
    const double alpha = s_alpha, nalpha = -alpha;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kDotThreads) {
        x[i] = __dadd_rn(__dmul_rn(1.0, x[i]), __dmul_rn(alpha, p[i]));
        const double rn = __dadd_rn(__dmul_rn(1.0, r[i]), __dmul_rn(nalpha, ap[i]));
        r[i] = rn;
        acc = __dadd_rn(acc, __dmul_rn(rn, rn));
    }
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < kDotThreads / 32 ? s[threadIdx.x] : 0.0;
        for (int o = 4; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
        if (threadIdx.x == 0) {
            partial[blockIdx.x] = acc;
            __threadfence();  // the partial sum before the ticket
            s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        }
    }
    __syncthreads();
    if (!s_last) return;
    // the last block: every other block has written its partial sum (and has read scal for the last time)
    __threadfence();
    const double rr = block_ordered_sum(partial, (int)gridDim.x, s_buf);
    if (threadIdx.x == 0) {
        *ticket = 0;
        const double rz_old = __ldcg(scal + 2), bnorm = __ldcg(scal + 6), tol = __ldcg(scal + 7);
        const double rel = sqrt(rr) / bnorm;  // ||r||2 / ||b||2
        const int it = (int)__ldcg(scal + 9) + 1;
        // [0] p.Ap [1] alpha [2] r.z [3] r.r [4] beta = r.z_new / r.z [5] stop [6] ||b|| [7] tolerance [8] ||r||/||b|| [9] iterations
        const double v[10] = {pap_sum, alpha, rr, rr, rr / rz_old, (!isfinite(alpha) || !isfinite(rel) || rel <= tol) ? 1.0 : 0.0,
                              bnorm,   tol,   rel, (double)it};
        double *rec = host_ring + (size_t)(it % ring_slots) * 16;
        for (int i = 0; i < 10; i++) scal[i] = v[i], rec[i] = v[i];
        __threadfence_system();
    }
}
// x = 1*x + alpha*p (waxpby 1), r = 1*r + (-alpha)*Ap (waxpby 2), partial sums of r.r (dots 2 and 3) in one pass
__global__ void __launch_bounds__(kDotThreads) cg_update_kernel(const double *__restrict__ scal, const double *__restrict__ p,
                                                               const double *__restrict__ ap, double *__restrict__ x,
                                                               double *__restrict__ r, int64_t n, double *__restrict__ partial) {
    __shared__ double s[kDotThreads / 32];
    if (scal[5] != 0.0) return;
    const double alpha = scal[1], nalpha = -alpha;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kDotThreads) {
        x[i] = __dadd_rn(__dmul_rn(1.0, x[i]), __dmul_rn(alpha, p[i]));
        const double rn = __dadd_rn(__dmul_rn(1.0, r[i]), __dmul_rn(nalpha, ap[i]));
        r[i] = rn;
        acc = __dadd_rn(acc, __dmul_rn(rn, rn));
    }
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < kDotThreads / 32 ? s[threadIdx.x] : 0.0;
        for (int o = 4; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
        if (threadIdx.x == 0) partial[blockIdx.x] = acc;
    }
}
// ... and the iteration's record of scalars goes straight into the host's pinned ring (slot = iteration number mod ring size;
// scal[9] counts the iterations), so that an iteration is kernels only and can be replayed as a CUDA graph
__global__ void cg_beta_kernel(const double *__restrict__ partial, int count, double *__restrict__ scal, double *host_ring, int ring_slots) {
    if (scal[5] != 0.0) return;
    __shared__ double s_buf[kSumChunk];
    const double acc = block_ordered_sum(partial, count, s_buf);
    if (threadIdx.x == 0) {
        const double rel = sqrt(acc) / scal[6];  // ||r||2 / ||b||2
        scal[3] = acc;
        scal[8] = rel;
        scal[4] = acc / scal[2];  // beta = r.z_new / r.z
        scal[2] = acc;
        if (!isfinite(scal[1]) || !isfinite(rel) || rel <= scal[7]) scal[5] = 1.0;
        const int it = (int)scal[9] + 1;
        scal[9] = (double)it;
        double *rec = host_ring + (size_t)(it % ring_slots) * 16;
        for (int i = 0; i < 10; i++) rec[i] = scal[i];
        __threadfence_system();
    }
}
// p = 1*r + beta*p (waxpby 3) with beta taken from the device
__global__ void cg_direction_kernel(const double *__restrict__ scal, const double *__restrict__ r, double *__restrict__ p, int64_t n) {
    pdl_launch_dependents();  // (no-ops unless launched with programmatic stream serialization)
    pdl_grid_dependency_wait();
    if (scal[5] != 0.0) return;
    const double beta = scal[4];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        p[i] = __dadd_rn(__dmul_rn(1.0, r[i]), __dmul_rn(beta, p[i]));
}

struct DotScratch {
    double *partial = nullptr, *out = nullptr, *scal = nullptr;
    double *partial2 = nullptr;       // r.r partial sums of the fused vector kernel (p.Ap's are still being read by other blocks)
    unsigned int *ticket = nullptr;   // its "last block" counter (zero between launches)
    ~DotScratch() {
        if (partial2) cudaFree(partial2);
        if (ticket) cudaFree(ticket);
        if (partial) cudaFree(partial);
        if (out) cudaFree(out);
        if (scal) cudaFree(scal);
    }
    int init() {
        SPMVB_CUDA(cudaMalloc(&partial, kPartialCap * sizeof(double)));
        SPMVB_CUDA(cudaMalloc(&out, sizeof(double)));
        SPMVB_CUDA(cudaMalloc(&scal, 16 * sizeof(double)));
        SPMVB_CUDA(cudaMalloc(&partial2, kPartialCap * sizeof(double)));
        SPMVB_CUDA(cudaMalloc(&ticket, sizeof(unsigned int)));
        SPMVB_CUDA(cudaMemset(ticket, 0, sizeof(unsigned int)));
        return SPMVB_OK;
    }
};

static int dot_device(const double *u, const double *v, int64_t n, DotScratch &sc, double *host, cudaStream_t st) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + kDotThreads - 1) / kDotThreads, kDotBlocks));
    dot_partial_kernel<<<blocks, kDotThreads, 0, st>>>(u, v, n, sc.partial);
    dot_final_kernel<<<1, 256, 0, st>>>(sc.partial, blocks, sc.out);
    SPMVB_CUDA(cudaMemcpyAsync(host, sc.out, sizeof(double), cudaMemcpyDeviceToHost, st));
    SPMVB_CUDA(cudaStreamSynchronize(st));
    return SPMVB_OK;
}

static int waxpby_device(double alpha, const double *x, double beta, const double *y, double *w, int64_t n, cudaStream_t st) {
    if (n <= 0) return SPMVB_OK;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, sm_count() * 16);
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
    // SPMVB_CG_TRACE=1: wall-clock of the phases of a solve on stderr (allocation, set-up, iterations, release)
    static const bool trace = std::getenv("SPMVB_CG_TRACE") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto t0, auto t1) { return std::chrono::duration<double, std::milli>(t1 - t0).count(); };
    const auto t_begin = now();
    auto t_alloc = t_begin, t_setup = t_begin, t_loop = t_begin;
    *iterations = 0;
    *converged = 0;
    // r, p, Ap: one block of 3 * n_pad doubles.  cudaMalloc / cudaFree of vectors this size cost ~1 ms each and now and then
    // 10-150 ms (measured, profiles/r01_cg_probe.log), so the block stays on the handle between solves ("cg_keep_workspace").
    const int64_t n_pad = (n + 63) / 64 * 64;
    DotScratch sc;
    SPMVB_TRY(sc.init());
    double *ws = nullptr;
    bool ws_on_handle = false;
    if (options().cg_keep_workspace && __atomic_exchange_n(&a->cg_ws_busy, 1, __ATOMIC_ACQUIRE) == 0) {
        ws_on_handle = true;
        if (!a->cg_ws && cudaMalloc(&a->cg_ws, (size_t)n_pad * 3 * sizeof(double)) != cudaSuccess) {
            a->cg_ws = nullptr;
            __atomic_store_n(&a->cg_ws_busy, 0, __ATOMIC_RELEASE);
            return fail(SPMVB_ERR_CUDA, "cg_solve: work vectors (%lld doubles): %s", (long long)n_pad * 3, cudaGetErrorString(cudaGetLastError()));
        }
        ws = a->cg_ws;
    } else if (cudaMalloc(&ws, (size_t)n_pad * 3 * sizeof(double)) != cudaSuccess) {
        return fail(SPMVB_ERR_CUDA, "cg_solve: work vectors (%lld doubles): %s", (long long)n_pad * 3, cudaGetErrorString(cudaGetLastError()));
    }
    double *r = ws, *p = ws + n_pad, *ap = ws + 2 * n_pad;
    int rc = SPMVB_OK;
    auto done = [&](int code) {
        if (trace) t_loop = now();
        if (ws_on_handle) {
            if (!options().cg_keep_workspace) {
                cudaFree(a->cg_ws);
                a->cg_ws = nullptr;
            }
            __atomic_store_n(&a->cg_ws_busy, 0, __ATOMIC_RELEASE);
        } else {
            cudaFree(ws);
        }
        if (trace)
            std::fprintf(stderr, "[spmvb cg] alloc %.3f ms, set-up %.3f ms, %d iterations %.3f ms, release %.3f ms\n", ms(t_begin, t_alloc),
                         ms(t_alloc, t_setup), *iterations, ms(t_setup, t_loop), ms(t_loop, now()));
        return code;
    };
    if (rc != SPMVB_OK) return done(rc);
    t_alloc = t_setup = now();
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
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + kDotThreads - 1) / kDotThreads, kDotBlocks));
    const int wblocks = (int)std::min<int64_t>((n + 255) / 256, sm_count() * 16);
    {
        const double init[16] = {0.0, 0.0, rz, 0.0, 0.0, 0.0, bnorm, tolerance, 0.0};
        // (every exit after the workspace was taken goes through done(): it releases or frees the work vectors)
        if (cudaMemcpyAsync(sc.scal, init, sizeof(init), cudaMemcpyHostToDevice, st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
            return done(fail(SPMVB_ERR_CUDA, "cg_solve: scalar set-up failed: %s", cudaGetErrorString(cudaGetLastError())));
    }
    // The host queues iteration `it` before it looks at the scalars of iteration it-kAhead (pinned ring of kRing records,
    // one event each): the stop decision is the device's (scal[5]); what was queued past it runs as no-ops (the SpMVs
    // still run, into the scratch vector).  kAhead iterations of queued work ride out a host thread that is descheduled
    // for a millisecond; with one iteration of run-ahead the device drained every time that happened.
    // (the pinned ring and the events are allocated once per host thread and device: cudaMallocHost costs milliseconds, and an
    // event or stream belongs to the device that was current when it was created)
    constexpr int kRing = 8, kAhead = 4;
    struct HostRing {
        double *ring = nullptr;
        cudaEvent_t ev[kRing] = {};
        int init() {
            if (ring) return SPMVB_OK;
            bool ok = cudaMallocHost(&ring, kRing * 16 * sizeof(double)) == cudaSuccess;
            for (int i = 0; ok && i < kRing; i++) ok = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) == cudaSuccess;
            if (!ok) {
                ring = nullptr;
                return fail(SPMVB_ERR_CUDA, "cg_solve: pinned scalar ring / events: %s", cudaGetErrorString(cudaGetLastError()));
            }
            return SPMVB_OK;
        }
    };
    static thread_local PerDevice<HostRing> hr_dev;
    HostRing &hr = hr_dev.get();
    if (hr.init() != SPMVB_OK) return done(SPMVB_ERR_CUDA);
    double *ring = hr.ring;
    cudaEvent_t *ev = hr.ev;
    auto finish = [&](int code) {
        cudaStreamSynchronize(st);
        return done(code);
    };
    // looks at iteration k (already queued); returns 1 to stop, 0 to go on, < 0 on error
    auto harvest = [&](int k) -> int {
        if (cudaEventSynchronize(ev[k % kRing]) != cudaSuccess) return -1;
        const double *h = ring + (k % kRing) * 16;
        const double alpha = h[1], rel = h[8];
        *iterations = k;
        if (residual_history) residual_history[k] = rel;
        if (!std::isfinite(alpha) || !std::isfinite(rel)) return 2;
        if (h[5] != 0.0) {
            *converged = 1;
            return 1;
        }
        return 0;
    };
    t_setup = now();
    int stop = 0, queued = 0, seen = 0;
    // One iteration, queued on `qs`: 1 SpMV (the pattern format's tensor-ring kernel also leaves the partial sums of p.Ap
    // when it can), dot 1 and alpha, waxpby 1 + 2 with dots 2 = 3, beta / stop flag / record, waxpby 3.
    bool fused_dot = false;
    auto queue_iteration = [&](cudaStream_t qs, bool direction) -> int {
        FusedDot fused{sc.partial, kPartialCap, 0};
        fused_dot_request() = options().cg_fused_dot ? &fused : nullptr;
        const int rc2 = spmvb_spmv(a, p, 0, n, ap, 0, (int32_t)n, qs);
        fused_dot_request() = nullptr;
        if (rc2 != SPMVB_OK) return rc2;
        fused_dot = fused.count != 0;
        if (!fused_dot) dot_partial_kernel<<<blocks, kDotThreads, 0, qs>>>(p, ap, n, sc.partial);
        if (options().cg_fused_scalars) {
            // one vector kernel: alpha at its head, beta / stop flag / record by its last block; it and the direction kernel are
            // launched with programmatic stream serialization (their blocks take the places of the previous kernel's as those exit)
            cudaLaunchAttribute pdl[1];
            pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            pdl[0].val.programmaticStreamSerializationAllowed = 1;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(blocks), cfg.blockDim = dim3(kDotThreads), cfg.stream = qs, cfg.attrs = pdl, cfg.numAttrs = options().cg_pdl ? 1 : 0;
            const double *pap = nullptr;
            int pap_count = 0;
            if (options().cg_fused_scalars == 2) pap = sc.partial, pap_count = fused_dot ? fused.count : blocks;  // alpha at the head of every block
            else cg_alpha_kernel<<<1, 256, 0, qs>>>(sc.partial, fused_dot ? fused.count : blocks, sc.scal);
            if (cudaLaunchKernelEx(&cfg, cg_update_fused_kernel, sc.scal, (const double *)p, (const double *)ap, x_dev, r, n, pap, pap_count,
                                   sc.partial2, sc.ticket, ring, (int)kRing) != cudaSuccess)
                return fail(SPMVB_ERR_CUDA, "cg_solve: launch failed: %s", cudaGetErrorString(cudaGetLastError()));
            if (direction) {
                cfg.gridDim = dim3(wblocks), cfg.blockDim = dim3(256);
                if (cudaLaunchKernelEx(&cfg, cg_direction_kernel, (const double *)sc.scal, (const double *)r, p, n) != cudaSuccess)
                    return fail(SPMVB_ERR_CUDA, "cg_solve: launch failed: %s", cudaGetErrorString(cudaGetLastError()));
            }
            return SPMVB_OK;
        }
        cg_alpha_kernel<<<1, 256, 0, qs>>>(sc.partial, fused_dot ? fused.count : blocks, sc.scal);
        cg_update_kernel<<<blocks, kDotThreads, 0, qs>>>(sc.scal, p, ap, x_dev, r, n, sc.partial);
        cg_beta_kernel<<<1, 256, 0, qs>>>(sc.partial, blocks, sc.scal, ring, kRing);
        if (direction) cg_direction_kernel<<<wblocks, 256, 0, qs>>>(sc.scal, r, p, n);
        return cudaGetLastError() == cudaSuccess ? SPMVB_OK : fail(SPMVB_ERR_CUDA, "cg_solve: launch failed");
    };
    // The first iteration is queued directly (it also completes every lazy set-up of the SpMV launch); the iteration is then
    // recorded once into a CUDA graph and replayed: one graph launch and one event per iteration on the host instead of
    // seven launches, which keeps a slow or busy host thread from starving the device ("cg_graph" = 0: direct launches).
    cudaGraphExec_t gexec = nullptr;
    auto finish_graph = [&](int code) {
        if (gexec) cudaGraphExecDestroy(gexec);
        return finish(code);
    };
    options().last_cg_graph = 0;
    for (int it = 1; it <= max_iterations && !stop; it++) {
        if (it == 2 && options().cg_graph && max_iterations > 2) {
            static thread_local PerDevice<cudaStream_t> cs_dev;
            cudaStream_t &cs = cs_dev.get();
            if (!cs && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) cs = nullptr;
            cudaGraph_t graph = nullptr;
            if (cs && cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
                const int rcq = queue_iteration(cs, true);
                const bool ended = cudaStreamEndCapture(cs, &graph) == cudaSuccess && graph;
                if (rcq != SPMVB_OK || !ended || cudaGraphInstantiate(&gexec, graph, nullptr, nullptr, 0) != cudaSuccess) gexec = nullptr;
                if (graph) cudaGraphDestroy(graph);
            }
            (void)cudaGetLastError();  // a failed capture leaves the direct launches
            options().last_cg_graph = gexec != nullptr;
        }
        if (gexec) {
            if (cudaGraphLaunch(gexec, st) != cudaSuccess) {
                finish_graph(SPMVB_OK);
                return fail(SPMVB_ERR_CUDA, "cg_solve: graph launch failed: %s", cudaGetErrorString(cudaGetLastError()));
            }
        } else {
            rc = queue_iteration(st, it < max_iterations);
            if (rc != SPMVB_OK) return finish_graph(rc);
        }
        options().last_cg_fused_dot = fused_dot;
        if (cudaEventRecord(ev[it % kRing], st) != cudaSuccess) {
            finish_graph(SPMVB_OK);
            return fail(SPMVB_ERR_CUDA, "cg_solve: %s", cudaGetErrorString(cudaGetLastError()));
        }
        queued = it;
        if (it > kAhead) stop = harvest(seen = it - kAhead);
    }
    while (!stop && seen < queued) stop = harvest(++seen);  // the last iterations queued (max_iterations reached)
    if (stop < 0 || cudaGetLastError() != cudaSuccess) {
        finish_graph(SPMVB_OK);
        return fail(SPMVB_ERR_CUDA, "cg_solve: device error in the iteration");
    }
    if (stop == 2) {
        const int at = *iterations;
        finish_graph(SPMVB_OK);
        return fail(SPMVB_ERR_DIVERGENCE, "cg_solve: non-finite value in iteration %d", at);  // inc/solver.hpp:44
    }
    return finish_graph(SPMVB_OK);
}

}  // extern "C"
