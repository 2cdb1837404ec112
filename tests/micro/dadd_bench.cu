// Microbenchmark: dependent-issue latency and throughput of DADD / DFMA on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o dadd_bench dadd_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS, bool FMA>
__global__ void chain_kernel(double *out, const double *in, int iters, long long *cycles) {
    double acc[CHAINS];
    double e[4];
    for (int i = 0; i < 4; i++) e[i] = in[i];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) acc[c] = in[4 + c];
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 16; k++) {
#pragma unroll
            for (int c = 0; c < CHAINS; c++) {
                if (FMA) acc[c] = __fma_rn(acc[c], e[(k + c) & 3], e[(k + c + 1) & 3]);
                else acc[c] = __dsub_rn(acc[c], e[(k + c) & 3]);
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

template <int CHAINS, bool FMA>
void run(int warps_per_block, int blocks) {
    double *out, *in;
    long long *cyc, h;
    cudaMalloc(&out, sizeof(double) * 1024 * 2048);
    cudaMalloc(&in, sizeof(double) * 64);
    cudaMalloc(&cyc, 8);
    double hin[64];
    for (int i = 0; i < 64; i++) hin[i] = 1.0 + i * 1e-3;
    cudaMemcpy(in, hin, sizeof hin, cudaMemcpyHostToDevice);
    const int iters = 2000;
    chain_kernel<CHAINS, FMA><<<blocks, warps_per_block * 32>>>(out, in, iters, cyc);
    chain_kernel<CHAINS, FMA><<<blocks, warps_per_block * 32>>>(out, in, iters, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)iters * 16 * CHAINS;  // per warp
    printf("%s chains/thread=%d warps/block=%2d blocks=%4d: %.2f cycles per op per warp; per-SM warp-ops/cycle = %.3f\n",
           FMA ? "DFMA" : "DADD", CHAINS, warps_per_block, blocks, h / ops, ops * warps_per_block * (blocks >= 148 ? (blocks / 148.0) : 1.0) / h);
    cudaFree(out); cudaFree(in); cudaFree(cyc);
}

int main() {
    run<1, false>(1, 1);
    run<2, false>(1, 1);
    run<4, false>(1, 1);
    run<8, false>(1, 1);
    run<1, true>(1, 1);
    run<4, false>(4, 1);
    run<4, false>(8, 1);
    run<4, false>(12, 1);
    run<4, false>(16, 1);
    run<8, false>(8, 1);
    run<8, false>(16, 148);
    run<4, false>(12, 148);
    run<8, true>(16, 148);
    return 0;
}
