// Device-side matrix generator: generate_matrix (inc/stencil.hpp:40-45,
// SPEC.md:48-56) for a range of global rows of the grid, with the optional
// config-4 perturbation (BASELINE.json configs[3]; recipe in DESIGN.md "C4 recipe").
// Output is a CSR handle (StencilMatrix layout, inc/stencil.hpp:19-36): row_start
// int64, cols int32 strictly ascending and GLOBAL, vals fp64.
#include <cub/cub.cuh>

#include "common.cuh"
#include "hash.cuh"

namespace spmvb {

constexpr int kMaxGenRow = 32;  // 27 stencil entries + up to 4 added

struct GenParams {
    int nx, ny, nz;
    int64_t n;  // global rows
    double diag, off;
    int perturb;
    uint64_t seed;
    double fraction, noise;
};

// Row of node (ix,iy,iz), row id = ix + nx*(iy + ny*iz) (inc/grid.hpp:13-14): couples
// to every in-grid (ix+dx,iy+dy,iz+dz); out-of-grid couplings omitted.
// Enumerating dz,dy,dx ascending yields strictly ascending columns.
__device__ int stencil_row(const GenParams &g, int64_t row, int32_t *cols, double *vals) {
    const int ix = (int)(row % g.nx);
    const int iy = (int)((row / g.nx) % g.ny);
    const int iz = (int)(row / ((int64_t)g.nx * g.ny));
    int k = 0;
    for (int dz = -1; dz <= 1; dz++) {
        const int z = iz + dz;
        if (z < 0 || z >= g.nz) continue;
        for (int dy = -1; dy <= 1; dy++) {
            const int y = iy + dy;
            if (y < 0 || y >= g.ny) continue;
            for (int dx = -1; dx <= 1; dx++) {
                const int x = ix + dx;
                if (x < 0 || x >= g.nx) continue;
                const int64_t c = x + (int64_t)g.nx * (y + (int64_t)g.ny * z);
                cols[k] = (int32_t)c;
                vals[k] = (c == row) ? g.diag : g.off;
                k++;
            }
        }
    }
    return k;
}

// Config-4 perturbation: a pure function of (seed, row).  A row is perturbed with
// probability `fraction`; 1..4 steps each drop one off-diagonal or add one absent
// in-range column; off-diagonals become off + (2u-1)*noise; the diagonal becomes
// the sum of |off-diagonal| (ascending column order) to keep weak dominance.
__device__ int perturb_row(const GenParams &g, int64_t row, int32_t *cols, double *vals, int k) {
    if (!(u01(h3(g.seed, (uint64_t)row, 0)) < g.fraction)) return k;
    const int steps = 1 + (int)(h3(g.seed, (uint64_t)row, 1) & 3);
    for (int s = 0; s < steps; s++) {
        const uint64_t hs = h3(g.seed, (uint64_t)row, 2 + (uint64_t)s);
        const int n_off = k - 1;
        const bool drop = ((hs & 1) == 0) && n_off > 0;
        if (drop) {
            const int j = (int)((hs >> 1) % (uint64_t)n_off);
            int pos = -1, seen = 0;
            for (int t = 0; t < k; t++) {
                if (cols[t] == row) continue;
                if (seen == j) { pos = t; break; }
                seen++;
            }
            for (int t = pos; t + 1 < k; t++) { cols[t] = cols[t + 1]; vals[t] = vals[t + 1]; }
            k--;
        } else {
            if ((int64_t)k >= g.n) continue;
            int64_t c = (int64_t)((hs >> 1) % (uint64_t)g.n);
            for (;;) {
                bool present = false;
                for (int t = 0; t < k; t++) if (cols[t] == c) { present = true; break; }
                if (!present) break;
                c = (c + 1) % g.n;
            }
            int pos = k;
            while (pos > 0 && cols[pos - 1] > c) { cols[pos] = cols[pos - 1]; vals[pos] = vals[pos - 1]; pos--; }
            cols[pos] = (int32_t)c;
            vals[pos] = g.off;
            k++;
        }
    }
    double sum = 0.0;
    int t_off = 0, dpos = -1;
    for (int t = 0; t < k; t++) {
        if (cols[t] == row) { dpos = t; continue; }
        const double u = u01(h3(g.seed, (uint64_t)row, 16 + (uint64_t)t_off));
        const double w = __dmul_rn(__dsub_rn(__dmul_rn(2.0, u), 1.0), g.noise);
        vals[t] = __dadd_rn(g.off, w);
        sum = __dadd_rn(sum, fabs(vals[t]));
        t_off++;
    }
    if (dpos >= 0) vals[dpos] = (t_off > 0) ? sum : g.diag;
    return k;
}

__device__ __forceinline__ int gen_row(const GenParams &g, int64_t row, int32_t *cols, double *vals) {
    int k = stencil_row(g, row, cols, vals);
    if (g.perturb) k = perturb_row(g, row, cols, vals, k);
    return k;
}

__global__ void gen_count_kernel(GenParams g, int64_t row_begin, int64_t nl, int64_t *counts) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nl) return;
    int32_t cols[kMaxGenRow];
    double vals[kMaxGenRow];
    counts[i] = gen_row(g, row_begin + i, cols, vals);
}

__global__ void gen_fill_kernel(GenParams g, int64_t row_begin, int64_t nl, const int64_t *__restrict__ row_start,
                                int32_t *__restrict__ out_cols, double *__restrict__ out_vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nl) return;
    int32_t cols[kMaxGenRow];
    double vals[kMaxGenRow];
    const int k = gen_row(g, row_begin + i, cols, vals);
    const int64_t b = row_start[i];
    for (int t = 0; t < k; t++) { out_cols[b + t] = cols[t]; out_vals[b + t] = vals[t]; }
}

int exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t count, cudaStream_t st) {
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    SPMVB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, in, out, count, st));
    SPMVB_CUDA(cudaMalloc(&tmp, tmp_bytes ? tmp_bytes : 16));
    cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, count, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(tmp);
    if (e != cudaSuccess) return fail(SPMVB_ERR_CUDA, "scan failed: %s", cudaGetErrorString(e));
    return SPMVB_OK;
}

}  // namespace spmvb

using namespace spmvb;

extern "C" int spmvb_generate_csr(const spmvb_grid *grid, int64_t row_begin, int64_t row_end, void *stream,
                                  spmvb_matrix **out) {
    if (!grid || !out) return fail(SPMVB_ERR_INVALID_ARGUMENT, "generate_csr: NULL argument");
    *out = nullptr;
    // inc/grid.hpp:35-47
    if (grid->nx < 1 || grid->ny < 1 || grid->nz < 1)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "grid dimensions must be >= 1, got %dx%dx%d", grid->nx, grid->ny, grid->nz);
    const double rows_d = (double)grid->nx * grid->ny * grid->nz;
    if (rows_d > 2147483647.0)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "grid %dx%dx%d has %.0f rows; column indices must fit a 4-byte signed integer",
                    grid->nx, grid->ny, grid->nz, rows_d);
    const int64_t n = (int64_t)grid->nx * grid->ny * grid->nz;
    if (row_begin < 0 || row_end > n || row_begin > row_end)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "row range [%lld,%lld) outside [0,%lld)", (long long)row_begin,
                    (long long)row_end, (long long)n);
    const int64_t nl = row_end - row_begin;
    cudaStream_t st = as_stream(stream);
    GenParams g{grid->nx, grid->ny, grid->nz, n, grid->diagonal, grid->off_diagonal, grid->perturb,
                grid->perturb_seed, grid->perturb_fraction, grid->perturb_noise};
    int dev = 0;
    SPMVB_CUDA(cudaGetDevice(&dev));
    spmvb_matrix *a = new spmvb_matrix();
    a->device = dev;
    a->format = SPMVB_FMT_CSR;
    a->n = (int32_t)nl;
    a->n_cols = n;
    a->row_offset = row_begin;
    int rc = dev_alloc(a, SPMVB_S_CSR_ROW_START, (uint64_t)(nl + 1) * 8);
    int64_t *counts = nullptr;
    if (rc == SPMVB_OK && cudaMalloc(&counts, (size_t)(nl + 1) * 8) != cudaSuccess) rc = fail(SPMVB_ERR_NOMEM, "out of device memory");
    const int threads = 128;
    const unsigned blocks = (unsigned)((nl + threads - 1) / threads);
    if (rc == SPMVB_OK) {
        cudaMemsetAsync(counts, 0, (size_t)(nl + 1) * 8, st);
        if (nl > 0) gen_count_kernel<<<blocks, threads, 0, st>>>(g, row_begin, nl, counts);
        rc = exclusive_scan_i64(counts, static_cast<int64_t *>(a->s[SPMVB_S_CSR_ROW_START]), nl + 1, st);
    }
    int64_t nnz = 0;
    if (rc == SPMVB_OK &&
        cudaMemcpy(&nnz, static_cast<int64_t *>(a->s[SPMVB_S_CSR_ROW_START]) + nl, 8, cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = fail(SPMVB_ERR_CUDA, "generate_csr: readback failed: %s", cudaGetErrorString(cudaGetLastError()));
    if (counts) cudaFree(counts);
    a->nnz = nnz;
    if (rc == SPMVB_OK) rc = dev_alloc(a, SPMVB_S_CSR_COLS, (uint64_t)nnz * 4);
    if (rc == SPMVB_OK) rc = dev_alloc(a, SPMVB_S_CSR_VALS, (uint64_t)nnz * 8);
    if (rc == SPMVB_OK && nl > 0) {
        gen_fill_kernel<<<blocks, threads, 0, st>>>(g, row_begin, nl, static_cast<const int64_t *>(a->s[SPMVB_S_CSR_ROW_START]),
                                                    static_cast<int32_t *>(a->s[SPMVB_S_CSR_COLS]),
                                                    static_cast<double *>(a->s[SPMVB_S_CSR_VALS]));
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = fail(SPMVB_ERR_CUDA, "generate_csr failed: %s", cudaGetErrorString(e));
    }
    if (rc != SPMVB_OK) { destroy(a); return rc; }
    *out = a;
    return SPMVB_OK;
}
