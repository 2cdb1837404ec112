// Data-movement skeleton of the pattern SpMV (no arithmetic): which march direction streams best?
//   mode Y: a warp owns 64 columns x 4 planes and marches over lines   (x box 68 x 1 line x 6 planes, ids 72 x 1 x 4)
//   mode Z: a warp owns 64 columns x 4 lines  and marches over planes  (x box 68 x 6 lines x 1 plane, ids 72 x 4 x 1)
// Per step and thread: wait for the set, read one value from it, store 8 rows of y.  4-slot ring per warp, CTA = 4 strips.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_march_bench tma_march_bench.cu && ./tma_march_bench 256 256 256
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            printf("%s failed: %s (line %d)\n", #x, cudaGetErrorString(e_), __LINE__); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

#ifndef RING_S
#define RING_S 4
#endif
#ifndef MINB
#define MINB 3
#endif
constexpr int S = RING_S, Q = 4, P = Q + 2;
constexpr uint32_t XB = 68 * 8 * P, XBP = (XB + 127) / 128 * 128, IB = 72 * 4 * Q, SLOT = XBP + (IB + 127) / 128 * 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\nWAIT_LOOP:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra DONE;\n\tbra WAIT_LOOP;\nDONE:\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap *tm, int c0, int c1, int c2, uint32_t bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
                 "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
                 : "memory");
}

// MODE 0 = Y march, 1 = Z march.  Work unit of a CTA: (group of 4 strips, block of Q planes [Y] / Q lines [Z]) x a range of
// march steps.  Units are enumerated with the unit index fastest across CTAs: blockIdx.x -> (unit, march chunk).
template <int MODE>
__global__ void __launch_bounds__(128, MINB)
    skeleton(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap ti, double *__restrict__ y, int sy, int pl, int np,
             int n_units, int chunk, int persistent, int total_steps, int do_store) {
    extern __shared__ unsigned char raw[];
    const uint32_t base = (smem_u32(raw) + 127u) & ~127u;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ring = base + warp * S * SLOT, bars = base + 4 * S * SLOT + warp * S * 8;
    // do_store == 2: y staged in shared memory (two buffers of Q x 512 B per warp) and written by bulk copies (aligned columns 64s .. 64s+63)
    const uint32_t stage = base + 4 * S * SLOT + 4 * S * 8 + 128 + warp * (2 * Q * 512);
    uint32_t n_st = 0;
    if (lane == 0) {
        for (int s = 0; s < S; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * s));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int n_sg = (sy + 255) / 256;
    const int march_len = MODE == 0 ? pl : np;
    const int64_t sz = (int64_t)sy * pl;
    uint32_t gs = 0;
    int pos, end;
    if (persistent) {  // equal contiguous chunks of the (unit-major) step sequence
        pos = blockIdx.x * chunk;
        end = min(total_steps, pos + chunk);
    } else {  // unit fastest across consecutive CTAs, chunk of the march per CTA
        const int unit = blockIdx.x % n_units, mc = blockIdx.x / n_units;
        pos = unit * march_len + mc * chunk;
        end = min(unit * march_len + march_len, pos + chunk);
    }
    double sink = 0.0;
    while (pos < end) {
        const int unit = pos / march_len, m0 = pos - unit * march_len, nb = min(march_len - m0, end - pos);
        const int strip = (unit % n_sg) * 4 + warp, blk = unit / n_sg;
        const int a_w = strip * 64 - 1;
        if (a_w < sy) {
            auto issue = [&](int k) {
                const uint32_t slot = (gs + k) % S, bar = bars + 8 * slot;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(XB + IB) : "memory");
                if (MODE == 0) {
                    tma3(ring + slot * SLOT, &tx, a_w - 1, m0 - 1 + k, blk * Q - 1, bar);
                    tma3(ring + slot * SLOT + XBP, &ti, a_w - 3, m0 - 1 + k, blk * Q, bar);
                } else {
                    tma3(ring + slot * SLOT, &tx, a_w - 1, blk * Q - 1, m0 - 1 + k, bar);
                    tma3(ring + slot * SLOT + XBP, &ti, a_w - 3, blk * Q, m0 - 1 + k, bar);
                }
            };
            const int n_sets = nb + 2;
            if (lane == 0)
                for (int k = 0; k < S && k < n_sets; k++) issue(k);
            mbar_wait(bars + 8 * (gs % S), (gs / S) & 1);
            mbar_wait(bars + 8 * ((gs + 1) % S), ((gs + 1) / S) & 1);
            const int a = a_w + 2 * lane;
            for (int j = 0; j < nb; j++) {
                mbar_wait(bars + 8 * ((gs + j + 2) % S), ((gs + j + 2) / S) & 1);
                double v;
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(ring + ((gs + j + 1) % S) * SLOT + lane * 16 + 8));
                if (do_store == 2) {
                    const uint32_t buf = stage + (n_st & 1) * (Q * 512);
                    if (n_st >= 2) {
                        if (lane < Q) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        __syncwarp();
                    }
#pragma unroll
                    for (int q = 0; q < Q; q++) asm volatile("st.shared.v2.f64 [%0], {%1,%2};" ::"r"(buf + q * 512 + lane * 16), "d"(v), "d"(v) : "memory");
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane < Q) {
                        const int q = lane;
                        const int64_t r = MODE == 0 ? (a_w + 1) + (int64_t)sy * (m0 + j) + sz * (blk * Q + q) : (a_w + 1) + (int64_t)sy * (blk * Q + q) + sz * (m0 + j);
                        const bool lok = MODE == 0 ? blk * Q + q < np : blk * Q + q < pl;
                        if (lok) asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(y + r), "r"(buf + q * 512) : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    n_st++;
                } else if (do_store) {
#pragma unroll
                    for (int q = 0; q < Q; q++) {
                        const int64_t r = MODE == 0 ? a + (int64_t)sy * (m0 + j) + sz * (blk * Q + q) : a + (int64_t)sy * (blk * Q + q) + sz * (m0 + j);
                        const bool lok = MODE == 0 ? blk * Q + q < np : blk * Q + q < pl;
                        if (lok && a >= 0) y[r] = v;
                        if (lok && a + 1 < sy) y[r + 1] = v;
                    }
                } else {
                    sink += v;
                }
                __syncwarp();
                if (lane == 0 && j + S < n_sets) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(j + S);
                }
            }
            gs += n_sets;
        }
        pos += nb;
        __syncwarp();
    }
    if (do_store == 2 && lane < Q) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (sink == 1.2345e-300) y[0] = sink;
}

using Enc = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                         const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
    const int sy = argc > 1 ? atoi(argv[1]) : 256, pl = argc > 2 ? atoi(argv[2]) : 256, np = argc > 3 ? atoi(argv[3]) : 256;
    const size_t n = (size_t)sy * pl * np;
    double *x, *y;
    int *ids;
    CK(cudaMalloc(&x, n * 8));
    CK(cudaMalloc(&y, n * 8));
    CK(cudaMalloc(&ids, n * 4));
    CK(cudaMemset(x, 0, n * 8));
    CK(cudaMemset(ids, 0, n * 4));
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
    Enc enc = reinterpret_cast<Enc>(fn);
    int n_sm = 0;
    CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0));
    const size_t smem = 4 * S * SLOT + 4 * S * 8 + 128 + 128 + 4 * 2 * Q * 512;
    for (int mode = 0; mode < 2; mode++) {
        CUtensorMap tx, ti;
        const cuuint64_t dims[3] = {(cuuint64_t)sy, (cuuint64_t)pl, (cuuint64_t)np};
        const cuuint64_t sx[2] = {(cuuint64_t)sy * 8, (cuuint64_t)sy * pl * 8}, si[2] = {(cuuint64_t)sy * 4, (cuuint64_t)sy * pl * 4};
        const cuuint32_t bx[3] = {68, (cuuint32_t)(mode ? P : 1), (cuuint32_t)(mode ? 1 : P)};
        const cuuint32_t bi[3] = {72, (cuuint32_t)(mode ? Q : 1), (cuuint32_t)(mode ? 1 : Q)};
        const cuuint32_t es[3] = {1, 1, 1};
        if (enc(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims, sx, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
            enc(&ti, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, ids, dims, si, bi, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed\n");
            return 1;
        }
        auto kern = mode ? skeleton<1> : skeleton<0>;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
        const int n_sg = (sy + 255) / 256;
        const int n_units = n_sg * ((mode ? pl : np) + Q - 1) / Q, march_len = mode ? np : pl;
        const int total = n_units * march_len;
        for (int store = 0; store < 3; store++)
            for (int sched = 0; sched < 6; sched++) {
                int persistent = sched == 0, chunk, grid;
                if (persistent) {
                    grid = n_sm * per_sm;
                    chunk = (total + grid - 1) / grid;
                } else {
                    const int chunks[] = {0, 8, 16, 32, 64, 1 << 30};
                    chunk = std::min(chunks[sched], march_len);
                    grid = n_units * ((march_len + chunk - 1) / chunk);
                }
                cudaEvent_t e0, e1;
                CK(cudaEventCreate(&e0));
                CK(cudaEventCreate(&e1));
                for (int w = 0; w < 3; w++) kern<<<grid, 128, smem>>>(tx, ti, y, sy, pl, np, n_units, chunk, persistent, total, store);
                CK(cudaEventRecord(e0));
                const int reps = 20;
                for (int w = 0; w < reps; w++) kern<<<grid, 128, smem>>>(tx, ti, y, sy, pl, np, n_units, chunk, persistent, total, store);
                CK(cudaEventRecord(e1));
                CK(cudaDeviceSynchronize());
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                const double us = ms * 1e3 / reps, bytes = (double)n * (store ? 20 : 12);
                printf("mode %c %-11s %s  grid %5d chunk %4d: %8.1f us  %7.1f GB/s algorithmic\n", mode ? 'Z' : 'Y', store == 2 ? "fetch+bulkst" : store ? "fetch+store" : "fetch only",
                       persistent ? "persistent" : "tiles     ", grid, chunk, us, bytes / us / 1e3);
            }
    }
    return 0;
}
