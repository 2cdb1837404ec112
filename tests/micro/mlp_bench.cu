// Microbenchmark: achieved HBM bandwidth of a read+write stream as a function of the bytes in
// flight per SM (warps per SM x independent 16-byte loads per thread), on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mlp_bench mlp_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void stream_kernel(const int4 *__restrict__ src, int4 *__restrict__ dst, size_t n_vec, int read_only) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    int4 acc = make_int4(0, 0, 0, 0);
    for (; i + (K - 1) * stride < n_vec; i += K * stride) {
        int4 v[K];
#pragma unroll
        for (int k = 0; k < K; k++) v[k] = src[i + k * stride];  // K independent loads in flight
        if (read_only) {
#pragma unroll
            for (int k = 0; k < K; k++) { acc.x ^= v[k].x; acc.y ^= v[k].y; acc.z ^= v[k].z; acc.w ^= v[k].w; }
        } else {
#pragma unroll
            for (int k = 0; k < K; k += 2) dst[(i + k * stride) / 2 + 0] = v[k];  // write half as much as is read (x+ids in, y out)
        }
    }
    if (read_only && acc.x == 0x12345678) dst[0] = acc;
}

template <int K>
void run(const int4 *src, int4 *dst, size_t n_vec, int ctas_per_sm, int threads, int read_only) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int grid = 148 * ctas_per_sm;
    stream_kernel<K><<<grid, threads>>>(src, dst, n_vec, read_only);
    cudaEventRecord(a);
    for (int r = 0; r < 5; r++) stream_kernel<K><<<grid, threads>>>(src, dst, n_vec, read_only);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    const double bytes = (double)n_vec * 16 * (read_only ? 1.0 : 1.5);
    const int warps = ctas_per_sm * threads / 32;
    printf("warps/SM %2d  K %2d  in flight/SM %6.1f KB  %s  %7.1f us  %6.2f TB/s\n", warps, K, warps * 32 * K * 16 / 1024.0,
           read_only ? "read " : "rd+wr", ms * 1e3, bytes / (ms * 1e-3) / 1e12);
}

int main() {
    const size_t n_vec = (size_t)1 << 26;  // 1 GiB of reads
    int4 *src, *dst;
    cudaMalloc(&src, n_vec * 16); cudaMalloc(&dst, n_vec * 16);
    cudaMemset(src, 1, n_vec * 16); cudaMemset(dst, 0, n_vec * 16);
    for (int ro = 1; ro >= 0; ro--) {
        for (int cps : {3, 4, 8, 16}) {
            run<1>(src, dst, n_vec, cps, 128, ro);
            run<2>(src, dst, n_vec, cps, 128, ro);
            run<4>(src, dst, n_vec, cps, 128, ro);
            run<8>(src, dst, n_vec, cps, 128, ro);
            run<16>(src, dst, n_vec, cps, 128, ro);
        }
    }
    return 0;
}
