// SpMV kernels for the row-major streams (ELL and value-table formats), sm_100a, fp64.
//
// Arithmetic contract: every product and every sum is rounded
// separately (__dmul_rn / __dadd_rn, never contracted to FMA), in the reference's documented
// per-format order (inc/kernels.hpp:19-22): bit-identical to the reference's loop built for
// baseline x86-64.
#include <algorithm>

#include "device_utils.cuh"
#include "spmv_internal.cuh"

namespace spmvb {

// ---- per-row accumulation from a staged tile (shared memory), reference order ---------------
// The gathers of x are issued in independent batches of B before the ordered sums consume
// them, so a row costs ~width/B L2 latencies instead of `width`.
template <int B>
__device__ __forceinline__ double ell_row(const double *v, const int32_t *c, int width, const double *__restrict__ x,
                                          int64_t x_col0) {
    // inc/kernels.hpp:19-20: slot order; padding slots multiply 0.0 by x[own row]
    double acc = 0.0;
    for (int base = 0; base < width; base += B) {
        double xv[B];
#pragma unroll
        for (int j = 0; j < B; j++) xv[j] = base + j < width ? __ldg(x + ((int64_t)c[base + j] - x_col0)) : 0.0;
#pragma unroll
        for (int j = 0; j < B; j++)
            if (base + j < width) acc = __dadd_rn(acc, __dmul_rn(v[base + j], xv[j]));
    }
    return acc;
}

template <int B>
__device__ __forceinline__ double vt_row(const int32_t *c, const int32_t *e, const double *tab, int m,
                                         const double *__restrict__ x, int64_t x_col0) {
    // inc/kernels.hpp:20-22: per value group (table order) sum x in stored order, then one product.
    // (Batching the gathers inside a group was measured slower than this plain loop: 509 vs 470 us
    // at 256^3 -- the group bookkeeping costs more than the latency it hides at full occupancy.)
    double acc = 0.0;
    int idx = 0;
    for (int k = 0; k < m; k++) {
        double sum = 0.0;
        const int end = e[k];
        for (; idx < end; idx++) sum = __dadd_rn(sum, __ldg(x + ((int64_t)c[idx] - x_col0)));
        acc = __dadd_rn(acc, __dmul_rn(tab[k], sum));
    }
    return acc;
}

// =============================================================================
// ELL (inc/ell.hpp:10-24; spmv: inc/kernels.hpp:23,31-32)
// Row-major n x width.  A tile of kTileRows rows is one contiguous block of each
// array; it is staged into shared memory with coalesced 128-bit loads, then each
// thread accumulates its own row in slot order (stride `width` doubles: conflict
// free for odd widths such as 27).  row_map != nullptr serves the exception block
// of the hybrid pattern format: tile rows are exception slots, y goes to row_map[e].
// =============================================================================
template <int ROWS, bool BULK = false, bool MAP = false>  // MAP: the exception block's own instantiation (row_map != nullptr), so that it can carry its own cache carve-out
__global__ void __launch_bounds__(ROWS) spmv_ell_kernel(const double *__restrict__ values,
                                                       const int32_t *__restrict__ columns, int width,
                                                       const double *__restrict__ x, int64_t x_col0,
                                                       double *__restrict__ y, int row_begin, int row_end,
                                                       int tile0, const int32_t *__restrict__ row_map, int n_rows) {
    extern __shared__ __align__(16) unsigned char smem[];
    double *sv = reinterpret_cast<double *>(smem);
    int32_t *sc = reinterpret_cast<int32_t *>(smem + (size_t)ROWS * width * 8);
    __shared__ __align__(8) uint64_t bar;
    const int r0 = (tile0 + blockIdx.x) * ROWS;
    const int64_t base = (int64_t)r0 * width;
    const int rows_here = min(ROWS, row_end - r0);
    const int nelem = rows_here * width;
    if (BULK && r0 + ROWS <= n_rows) {  // a whole tile by two bulk copies (see spmv_vt_kernel); co-resident CTAs overlap one another
        if (threadIdx.x == 0) {
            mbar_init(smem_u32(&bar), 1);
            fence_mbar_init();
            const uint32_t bytes_v = (uint32_t)ROWS * width * 8, bytes_c = (uint32_t)ROWS * width * 4;
            mbar_expect_tx(smem_u32(&bar), bytes_v + bytes_c);
            bulk_g2s(smem_u32(sv), values + base, bytes_v, smem_u32(&bar));
            bulk_g2s(smem_u32(sc), columns + base, bytes_c, smem_u32(&bar));
        }
        __syncthreads();
        mbar_wait(smem_u32(&bar), 0);
    } else {
        const int4 *gv = reinterpret_cast<const int4 *>(values + base);
        const int nv = (nelem + 1) >> 1;
#pragma unroll 4
        for (int i = threadIdx.x; i < nv; i += ROWS) reinterpret_cast<int4 *>(sv)[i] = ld_stream(gv + i);
        const int4 *gc = reinterpret_cast<const int4 *>(columns + base);
        const int nc = (nelem + 3) >> 2;
#pragma unroll 4
        for (int i = threadIdx.x; i < nc; i += ROWS) reinterpret_cast<int4 *>(sc)[i] = ld_stream(gc + i);
        __syncthreads();
    }
    const int r = r0 + threadIdx.x;
    if (r < row_begin || r >= row_end) return;
    const double *v = sv + threadIdx.x * width;
    const int32_t *c = sc + threadIdx.x * width;
    // exception block (row_map): its gathers mostly miss L1 (the rows are scattered), so all of a row's operands are requested at
    // once -- one L2 round trip per row instead of four
    if (row_map) y[row_map[r]] = (BULK && width <= 32) ? ell_row<32>(v, c, width, x, x_col0) : ell_row<9>(v, c, width, x, x_col0);
    else y[r] = (BULK && width == 27) ? ell_row<27>(v, c, 27, x, x_col0) : ell_row<9>(v, c, width, x, x_col0);
}

// Naive thread-per-row form, the A/B baseline ("ell_kernel" = 1; lab builds only, the default build runs its default kernel instead).
#ifdef SPMVB_LAB
__global__ void spmv_ell_naive_kernel(const double *__restrict__ values, const int32_t *__restrict__ columns,
                                      int width, const double *__restrict__ x, int64_t x_col0,
                                      double *__restrict__ y, int row_begin, int row_end) {
    const int r = row_begin + blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= row_end) return;
    const double *v = values + (int64_t)r * width;
    const int32_t *c = columns + (int64_t)r * width;
    double acc = 0.0;
    for (int k = 0; k < width; k++) acc = __dadd_rn(acc, __dmul_rn(v[k], __ldg(x + ((int64_t)c[k] - x_col0))));
    y[r] = acc;
}
#endif

// =============================================================================
// Value table (inc/compress.hpp:28-44; spmv: inc/kernels.hpp:24,33-34;
// SPEC.md:218-221): per row, sum x within each value group in stored order, then
// one product per group in table order.
// =============================================================================
template <int ROWS, bool BULK>
__global__ void __launch_bounds__(ROWS) spmv_vt_kernel(const int32_t *__restrict__ sorted_columns,
                                                      const int32_t *__restrict__ ends,
                                                      const double *__restrict__ table, int width, int m,
                                                      const double *__restrict__ x, int64_t x_col0,
                                                      double *__restrict__ y, int row_begin, int row_end,
                                                      int tile0, int n_rows) {
    extern __shared__ __align__(16) unsigned char smem[];
    int32_t *sc = reinterpret_cast<int32_t *>(smem);
    int32_t *se = sc + (size_t)ROWS * width;
    double *st = reinterpret_cast<double *>(se + (size_t)ROWS * m);
    __shared__ __align__(8) uint64_t bar;
    const int r0 = (tile0 + blockIdx.x) * ROWS;
    const int rows_here = min(ROWS, row_end - r0);
    // BULK: a whole tile is fetched by two bulk copies (cp.async.bulk, one elected thread) instead of 128-bit loads and
    // stores by every thread: the load/store unit is this kernel's busiest pipe (27 index reads + 27 gathers per row),
    // and the staging traffic was 40 % of its wavefronts.  Tiles that are not whole (the stream's last) keep the loads.
    const bool bulk = BULK && r0 + ROWS <= n_rows;
    if (bulk) {
        if (threadIdx.x == 0) {
            mbar_init(smem_u32(&bar), 1);
            fence_mbar_init();
            const uint32_t bytes_c = (uint32_t)ROWS * width * 4, bytes_e = (uint32_t)ROWS * m * 4;
            mbar_expect_tx(smem_u32(&bar), bytes_c + bytes_e);
            bulk_g2s(smem_u32(sc), sorted_columns + (int64_t)r0 * width, bytes_c, smem_u32(&bar));
            bulk_g2s(smem_u32(se), ends + (int64_t)r0 * m, bytes_e, smem_u32(&bar));
        }
        for (int i = threadIdx.x; i < m; i += ROWS) st[i] = table[i];
        __syncthreads();  // the barrier is initialised (and the table staged) before anyone waits on it
        mbar_wait(smem_u32(&bar), 0);
    } else {
        const int4 *gc = reinterpret_cast<const int4 *>(sorted_columns + (int64_t)r0 * width);
        const int nc = (rows_here * width + 3) >> 2;
#pragma unroll 4
        for (int i = threadIdx.x; i < nc; i += ROWS) reinterpret_cast<int4 *>(sc)[i] = ld_stream(gc + i);
        const int4 *ge = reinterpret_cast<const int4 *>(ends + (int64_t)r0 * m);
        const int ne = (rows_here * m + 3) >> 2;
        for (int i = threadIdx.x; i < ne; i += ROWS) reinterpret_cast<int4 *>(se)[i] = ld_stream(ge + i);
        for (int i = threadIdx.x; i < m; i += ROWS) st[i] = table[i];
        __syncthreads();
    }
    const int r = r0 + threadIdx.x;
    if (r < row_begin || r >= row_end) return;
    y[r] = vt_row<9>(sc + threadIdx.x * width, se + threadIdx.x * m, st, m, x, x_col0);
}

// =============================================================================
// TMA (bulk-copy) pipelines for the row-major streams.  A persistent CTA walks
// 128-row tiles; one elected thread issues `cp.async.bulk` (SASS UBLKCP) copies of
// the tile's contiguous value / column blocks into a ring of NS shared-memory
// stages, completion is signalled on an mbarrier per stage (complete_tx), all
// threads then accumulate their own row from shared memory in the reference
// order.  While one stage is consumed the other NS-1 are in flight, so HBM never
// idles during the gather/accumulate phase (the vectorised-load kernels above
// alternate between a load phase and a compute phase).
// =============================================================================
// FMT 0: ELL (a = values f64, b = columns i32, wa = wb = width)
// FMT 1: vt  (a unused,       b = sorted_columns i32 (wb = width), c = ends i32 (wc = m), table)
template <int ROWS, int NS, int FMT>
__global__ void __launch_bounds__(ROWS) spmv_rows_tma_kernel(const double *__restrict__ values,
                                                            const int32_t *__restrict__ columns,
                                                            const int32_t *__restrict__ ends,
                                                            const double *__restrict__ table, int width, int m,
                                                            const double *__restrict__ x, int64_t x_col0,
                                                            double *__restrict__ y, int row_begin, int row_end, int tile0,
                                                            int n_tiles, const int32_t *__restrict__ row_map) {
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t bytes_v = FMT == 0 ? (uint32_t)ROWS * width * 8 : 0;
    const uint32_t bytes_c = (uint32_t)ROWS * width * 4;
    const uint32_t bytes_e = FMT == 1 ? (uint32_t)ROWS * m * 4 : 0;
    const uint32_t stage_bytes = bytes_v + bytes_c + bytes_e;  // each a multiple of 16
    __shared__ __align__(8) uint64_t full_bar[NS];
    __shared__ double s_table[FMT == 1 ? 256 : 1];
    if (FMT == 1)
        for (int i = threadIdx.x; i < m && i < 256; i += ROWS) s_table[i] = table[i];
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; s++) mbar_init(smem_u32(&full_bar[s]), 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int it) {  // elected thread: fetch the it-th tile of this CTA into stage it % NS
        const int tile = blockIdx.x + it * gridDim.x;
        if (tile >= n_tiles) return;
        const int s = it % NS;
        const int64_t r0 = (int64_t)(tile0 + tile) * ROWS;
        const uint32_t bar = smem_u32(&full_bar[s]);
        const uint32_t dst = smem_u32(smem + (size_t)s * stage_bytes);
        mbar_expect_tx(bar, stage_bytes);
        if (FMT == 0) bulk_g2s(dst, values + r0 * width, bytes_v, bar);
        bulk_g2s(dst + bytes_v, columns + r0 * width, bytes_c, bar);
        if (FMT == 1) bulk_g2s(dst + bytes_v + bytes_c, ends + r0 * m, bytes_e, bar);
    };
    if (threadIdx.x == 0)
        for (int it = 0; it < NS; it++) issue(it);
    for (int it = 0;; it++) {
        const int tile = blockIdx.x + it * gridDim.x;
        if (tile >= n_tiles) break;
        const int s = it % NS;
        mbar_wait(smem_u32(&full_bar[s]), (it / NS) & 1);
        const unsigned char *st = smem + (size_t)s * stage_bytes;
        const int r = (tile0 + tile) * ROWS + threadIdx.x;
        if (r >= row_begin && r < row_end) {
            const int32_t *c = reinterpret_cast<const int32_t *>(st + bytes_v) + threadIdx.x * width;
            double acc;
            if (FMT == 0) {
                const double *v = reinterpret_cast<const double *>(st) + threadIdx.x * width;
                acc = width == 27 ? ell_row<27>(v, c, 27, x, x_col0) : ell_row<9>(v, c, width, x, x_col0);
            } else {
                const int32_t *e = reinterpret_cast<const int32_t *>(st + bytes_v + bytes_c) + threadIdx.x * m;
                const double *tab = m <= 256 ? s_table : table;
                acc = vt_row<9>(c, e, tab, m, x, x_col0);
            }
            y[row_map ? row_map[r] : r] = acc;
        }
        __syncthreads();  // every thread is done with stage s
        if (threadIdx.x == 0) {
            fence_proxy_async();  // order the generic-proxy reads before the async-proxy refill
            issue(it + NS);
        }
    }
}

// ---- host-side launchers -----------------------------------------------------------
int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SPMVB_ERR_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
    return SPMVB_OK;
}

int launch_ell(const double *values, const int32_t *columns, int width, const double *x, int64_t x_col0,
                      double *y, int row_begin, int row_end, const int32_t *row_map, cudaStream_t st) {
    if (row_end <= row_begin || width == 0) {
        if (width == 0 && row_end > row_begin && !row_map)
            SPMVB_CUDA(cudaMemsetAsync(y + row_begin, 0, (size_t)(row_end - row_begin) * 8, st));
        return SPMVB_OK;
    }
#ifdef SPMVB_LAB
    if (options().ell_kernel == 1 && !row_map) {
        const int threads = 128;
        spmv_ell_naive_kernel<<<(row_end - row_begin + threads - 1) / threads, threads, 0, st>>>(
            values, columns, width, x, x_col0, y, row_begin, row_end);
        return check_launch("spmv_ell_naive");
    }
#endif
    const int tile0 = row_begin / kTileRows;
    const int tiles = (row_end + kTileRows - 1) / kTileRows - tile0;
    const size_t smem = (size_t)kTileRows * width * 12;
    if (smem > 200 * 1024) return fail(SPMVB_ERR_INVALID_ARGUMENT, "ELL width %d too large for the staged kernel", width);
    {
        // One bulk-copied tile per CTA, many CTAs per SM.  Default: 32-row tiles (one warp per CTA, 10.4 KB at width 27, ~21
        // CTAs/SM): 795 us at 256^3 = 7.17 TB/s of algorithmic traffic -- a read-dominated stream, above the copy kernel's 6.54
        // TB/s (half reads, half writes).  64-row tiles 922 us, 128-row tiles 946 us (ell_kernel = 5, 4;
        // profiles/r01_probe256_ell_vt_bulk_tiles.log).  The persistent two-stage ring below (ell_kernel = 3) holds 2 CTAs/SM: 1021-1038 us.
        const int k = options().ell_kernel;
        const int rows = !kLabBuild ? 32 : k == 4 ? 128 : k == 5 ? 64 : 32;
        if ((k == 0 || (kLabBuild && (k == 4 || k == 5 || k == 6))) && (size_t)rows * width * 12 <= 200 * 1024) {
            static PerDevice<bool> attr;
            if (!attr.get()) {
#ifdef SPMVB_LAB
                SPMVB_CUDA(cudaFuncSetAttribute(spmv_ell_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                SPMVB_CUDA(cudaFuncSetAttribute(spmv_ell_kernel<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
#endif
                SPMVB_CUDA(cudaFuncSetAttribute(spmv_ell_kernel<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                attr.get() = true;
            }
            const int t0 = row_begin / rows, nt = (row_end + rows - 1) / rows - t0;
            const size_t bytes = (size_t)rows * width * 12;
            // whole tiles below row_end are bulk-copied; the last, partial one is staged with loads
#ifdef SPMVB_LAB
            if (rows == 128) spmv_ell_kernel<128, true><<<nt, 128, bytes, st>>>(values, columns, width, x, x_col0, y, row_begin, row_end, t0, row_map, row_end);
            else if (rows == 64) spmv_ell_kernel<64, true><<<nt, 64, bytes, st>>>(values, columns, width, x, x_col0, y, row_begin, row_end, t0, row_map, row_end);
            else
#endif
            if (row_map) {
                static PerDevice<int> map_attr;
                // The block's gathers are scattered (its rows are one grid row in ten), and what they hit in L1 they need not fetch
                // from L2: with the driver's carve-out 17 CTAs of 12.9 KB leave ~30 KB of L1 per SM; 60 % of the SM's 228 KB for
                // shared memory keeps 10 CTAs and 90 KB of L1 (block alone 34 -> 25-28 us, C4 overlapped 41.6 -> 38.8 us at 128^3;
                // 35 % and below starve the kernel of CTAs).  "exception_carveout": percent, 0 = this default, -1 = the driver's.
                const int opt = options().exception_carveout, carve = opt == 0 ? 60 : opt;
                if (map_attr.get() != carve + 1) {
                    SPMVB_CUDA(cudaFuncSetAttribute(spmv_ell_kernel<32, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                    SPMVB_CUDA(cudaFuncSetAttribute(spmv_ell_kernel<32, true, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                    carve > 0 ? carve : (int)cudaSharedmemCarveoutDefault));
                    map_attr.get() = carve + 1;
                }
                spmv_ell_kernel<32, true, true><<<nt, 32, bytes, st>>>(values, columns, width, x, x_col0, y, row_begin, row_end, t0, row_map, row_end);
            } else
            spmv_ell_kernel<32, true><<<nt, 32, bytes, st>>>(values, columns, width, x, x_col0, y, row_begin, row_end, t0, row_map, row_end);
            return check_launch("spmv_ell_bulk");
        }
    }
    if (options().ell_kernel != 2) {
        // persistent TMA bulk pipeline (ell_kernel = 3, and widths whose tile does not fit above): NS stages of one tile each
        constexpr int NS = 2;
        const size_t stage = smem;  // multiple of 16 for any width (128 rows)
        const size_t need = stage * NS;
        if (need <= 220 * 1024) {
            static PerDevice<bool> tma_attr;
            if (!tma_attr.get()) {
                SPMVB_CUDA(cudaFuncSetAttribute(spmv_rows_tma_kernel<kTileRows, NS, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
                tma_attr.get() = true;
            }
            const int per_sm = std::max(1, (int)std::min<size_t>(8, (220 * 1024) / (need + 1024)));
            const int grid = std::min(tiles, sm_count() * per_sm);
            spmv_rows_tma_kernel<kTileRows, NS, 0><<<grid, kTileRows, need, st>>>(values, columns, nullptr, nullptr, width, 0, x, x_col0, y,
                                                                               row_begin, row_end, tile0, tiles, row_map);
            return check_launch("spmv_ell_tma");
        }
    }
    static PerDevice<bool> attr_set;
    if (!attr_set.get()) {
        SPMVB_CUDA(cudaFuncSetAttribute(spmv_ell_kernel<kTileRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_set.get() = true;
    }
    spmv_ell_kernel<kTileRows><<<tiles, kTileRows, smem, st>>>(values, columns, width, x, x_col0, y, row_begin,
                                                               row_end, tile0, row_map, 0);
    return check_launch("spmv_ell");
}

int launch_vt(const spmvb_matrix *a, const double *x, int64_t x_col0, double *y, int row_begin, int row_end,
                     cudaStream_t st) {
    if (row_end <= row_begin) return SPMVB_OK;
    const int tile0 = row_begin / kTileRows;
    const int tiles = (row_end + kTileRows - 1) / kTileRows - tile0;
    const size_t smem = (size_t)kTileRows * (a->width + a->m) * 4 + (size_t)a->m * 8 + 16;
    if (smem > 200 * 1024) return fail(SPMVB_ERR_INVALID_ARGUMENT, "vt width/table too large for the staged kernel");
#ifdef SPMVB_LAB
    if (options().ell_kernel == 3) {  // TMA bulk pipeline: measured slower than the staged kernel for vt (545 vs 470 us); lab builds only
        constexpr int NS = 2;
        const size_t stage = (size_t)kTileRows * (a->width + a->m) * 4;
        const size_t need = stage * NS;
        if (need <= 200 * 1024) {
            static PerDevice<bool> tma_attr;
            if (!tma_attr.get()) {
                SPMVB_CUDA(cudaFuncSetAttribute(spmv_rows_tma_kernel<kTileRows, NS, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                tma_attr.get() = true;
            }
            const int per_sm = std::max(1, (int)std::min<size_t>(8, (200 * 1024) / (need + 4096)));
            const int grid = std::min(tiles, sm_count() * per_sm);
            spmv_rows_tma_kernel<kTileRows, NS, 1><<<grid, kTileRows, need, st>>>(
                nullptr, static_cast<const int32_t *>(a->s[SPMVB_S_SORTED_COLUMNS]), static_cast<const int32_t *>(a->s[SPMVB_S_ENDS]),
                static_cast<const double *>(a->s[SPMVB_S_TABLE]), a->width, a->m, x, x_col0, y, row_begin, row_end, tile0, tiles, nullptr);
            return check_launch("spmv_vt_tma");
        }
    }
#endif
    // bulk-copy staging needs 16-byte multiples per tile part: 128 rows x width (and x m) ints always are
    const bool bulk = options().ell_kernel != 2;
    static PerDevice<bool> attr_set;
    if (!attr_set.get()) {
        SPMVB_CUDA(cudaFuncSetAttribute(spmv_vt_kernel<kTileRows, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        SPMVB_CUDA(cudaFuncSetAttribute(spmv_vt_kernel<kTileRows, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_set.get() = true;
    }
    const auto *sc = static_cast<const int32_t *>(a->s[SPMVB_S_SORTED_COLUMNS]);
    const auto *se = static_cast<const int32_t *>(a->s[SPMVB_S_ENDS]);
    const auto *tab = static_cast<const double *>(a->s[SPMVB_S_TABLE]);
#ifdef SPMVB_LAB
    if (options().ell_kernel == 6) {  // 64-row tiles
        const int t0 = row_begin / 64, nt = (row_end + 63) / 64 - t0;
        static PerDevice<bool> a64;
        if (!a64.get()) {
            SPMVB_CUDA(cudaFuncSetAttribute(spmv_vt_kernel<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            a64.get() = true;
        }
        spmv_vt_kernel<64, true><<<nt, 64, (size_t)64 * (a->width + a->m) * 4 + (size_t)a->m * 8 + 16, st>>>(sc, se, tab, a->width, a->m, x, x_col0, y, row_begin, row_end, t0, a->n);
    } else if (options().ell_kernel == 7) {  // 32-row tiles
        const int t0 = row_begin / 32, nt = (row_end + 31) / 32 - t0;
        spmv_vt_kernel<32, true><<<nt, 32, (size_t)32 * (a->width + a->m) * 4 + (size_t)a->m * 8 + 16, st>>>(sc, se, tab, a->width, a->m, x, x_col0, y, row_begin, row_end, t0, a->n);
    } else
#endif
    if (bulk) spmv_vt_kernel<kTileRows, true><<<tiles, kTileRows, smem, st>>>(sc, se, tab, a->width, a->m, x, x_col0, y, row_begin, row_end, tile0, a->n);
    else spmv_vt_kernel<kTileRows, false><<<tiles, kTileRows, smem, st>>>(sc, se, tab, a->width, a->m, x, x_col0, y, row_begin, row_end, tile0, a->n);
    return check_launch("spmv_vt");
}

}  // namespace spmvb
