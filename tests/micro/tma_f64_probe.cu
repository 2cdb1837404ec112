// Probe: 3-D TMA tensor load of fp64 boxes {W,1,P} with negative / out-of-range coordinates (zero fill).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_f64_probe tma_f64_probe.cu && ./tma_f64_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap tm, double *out, int W, int P, int c0, int c1, int c2) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sb = ((uint32_t)__cvta_generic_to_shared(smem) + 127u) & ~127u;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(W * P * 8) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sb),
            "l"(&tm), "r"(c0), "r"(c1), "r"(c2), "r"(b)
            : "memory");
    }
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(b) : "memory");
    const double *s = reinterpret_cast<const double *>(smem + (sb - (uint32_t)__cvta_generic_to_shared(smem)));
    for (int i = threadIdx.x; i < W * P; i += blockDim.x) out[i] = s[i];
}

int main() {
    const int sy = 128, pl = 10, np = 6;
    const size_t n = (size_t)sy * pl * np;
    std::vector<double> h(n);
    for (size_t i = 0; i < n; i++) h[i] = (double)i + 0.5;
    double *x, *out;
    cudaMalloc(&x, n * 8);
    cudaMalloc(&out, 1 << 16);
    cudaMemcpy(x, h.data(), n * 8, cudaMemcpyHostToDevice);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
    for (int W : {64, 66, 34, 2}) {
        for (int dtype = 0; dtype < 2; dtype++) {  // 0: FLOAT64 elements; 1: the same bytes as pairs of 32-bit words
            const int P = 4;
            CUtensorMap tm;
            cuuint64_t dims[3] = {(cuuint64_t)(dtype ? sy * 2 : sy), pl, np};
            cuuint64_t strides[2] = {(cuuint64_t)sy * 8, (cuuint64_t)sy * pl * 8};
            cuuint32_t box[3] = {(cuuint32_t)(dtype ? W * 2 : W), 1, (cuuint32_t)P};
            cuuint32_t es[3] = {1, 1, 1};
            CUresult r = enc(&tm, dtype ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            printf("W=%d dtype=%s encode=%d\n", W, dtype ? "u32x2" : "f64", (int)r);
            if (r != CUDA_SUCCESS) continue;
            for (int c0 : {0, -1, sy - 3}) {
                const int c1 = 2, c2 = -1;
                cudaMemset(out, 0xff, 1 << 16);
                probe<<<1, 128, 16384>>>(tm, out, W, P, dtype ? c0 * 2 : c0, c1, c2);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("  c0=%d: %s\n", c0, cudaGetErrorString(e));
                    return 1;
                }
                std::vector<double> o((size_t)W * P);
                cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
                int bad = 0;
                for (int pz = 0; pz < P; pz++)
                    for (int i = 0; i < W; i++) {
                        const int a = c0 + i, c = c2 + pz;
                        const double want = (a < 0 || a >= sy || c < 0 || c >= np) ? 0.0 : h[(size_t)a + (size_t)sy * c1 + (size_t)sy * pl * c];
                        if (o[(size_t)pz * W + i] != want) bad++;
                    }
                printf("  c0=%d: %d mismatches of %d\n", c0, bad, W * P);
            }
        }
    }
    return 0;
}
