// SpMV kernels for sm_100a: y = A x, fp64, decompression fused into the product.
//
// Arithmetic contract: every product and every sum is
// rounded separately (__dmul_rn / __dadd_rn, never contracted to FMA), in the
// reference's documented per-format order (inc/kernels.hpp:19-22), so results are
// bit-identical to the reference's `y[i] += a_ij * x_j` built for baseline x86-64.
// Multiplication by -1.0 is exact, so `acc + (-1.0 * x)` is issued as `acc - x`.
#include <algorithm>

#include "common.cuh"

namespace spmvb {

// ---- streaming loads: read-once matrix data bypasses L1 allocation ---------------
__device__ __forceinline__ int4 ld_stream(const int4 *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ int ld_stream(const int *p) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// TMA-engine L2 prefetch of a contiguous range (address 16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void prefetch_l1(const void *p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}


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
template <int ROWS>
__global__ void __launch_bounds__(ROWS) spmv_ell_kernel(const double *__restrict__ values,
                                                       const int32_t *__restrict__ columns, int width,
                                                       const double *__restrict__ x, int64_t x_col0,
                                                       double *__restrict__ y, int row_begin, int row_end,
                                                       int tile0, const int32_t *__restrict__ row_map) {
    extern __shared__ __align__(16) unsigned char smem[];
    double *sv = reinterpret_cast<double *>(smem);
    int32_t *sc = reinterpret_cast<int32_t *>(smem + (size_t)ROWS * width * 8);
    const int r0 = (tile0 + blockIdx.x) * ROWS;
    const int64_t base = (int64_t)r0 * width;
    const int rows_here = min(ROWS, row_end - r0);
    const int nelem = rows_here * width;
    {
        const int4 *gv = reinterpret_cast<const int4 *>(values + base);
        const int nv = (nelem + 1) >> 1;
#pragma unroll 4
        for (int i = threadIdx.x; i < nv; i += ROWS) reinterpret_cast<int4 *>(sv)[i] = ld_stream(gv + i);
        const int4 *gc = reinterpret_cast<const int4 *>(columns + base);
        const int nc = (nelem + 3) >> 2;
#pragma unroll 4
        for (int i = threadIdx.x; i < nc; i += ROWS) reinterpret_cast<int4 *>(sc)[i] = ld_stream(gc + i);
    }
    __syncthreads();
    const int r = r0 + threadIdx.x;
    if (r < row_begin || r >= row_end) return;
    y[row_map ? row_map[r] : r] = ell_row<9>(sv + threadIdx.x * width, sc + threadIdx.x * width, width, x, x_col0);
}

// Naive thread-per-row form, kept as the A/B baseline ("ell_kernel" = 1).
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

// =============================================================================
// Value table (inc/compress.hpp:28-44; spmv: inc/kernels.hpp:24,33-34;
// SPEC.md:218-221): per row, sum x within each value group in stored order, then
// one product per group in table order.
// =============================================================================
template <int ROWS>
__global__ void __launch_bounds__(ROWS) spmv_vt_kernel(const int32_t *__restrict__ sorted_columns,
                                                      const int32_t *__restrict__ ends,
                                                      const double *__restrict__ table, int width, int m,
                                                      const double *__restrict__ x, int64_t x_col0,
                                                      double *__restrict__ y, int row_begin, int row_end,
                                                      int tile0) {
    extern __shared__ __align__(16) unsigned char smem[];
    int32_t *sc = reinterpret_cast<int32_t *>(smem);
    int32_t *se = sc + (size_t)ROWS * width;
    double *st = reinterpret_cast<double *>(se + (size_t)ROWS * m);
    const int r0 = (tile0 + blockIdx.x) * ROWS;
    const int rows_here = min(ROWS, row_end - r0);
    {
        const int4 *gc = reinterpret_cast<const int4 *>(sorted_columns + (int64_t)r0 * width);
        const int nc = (rows_here * width + 3) >> 2;
#pragma unroll 4
        for (int i = threadIdx.x; i < nc; i += ROWS) reinterpret_cast<int4 *>(sc)[i] = ld_stream(gc + i);
        const int4 *ge = reinterpret_cast<const int4 *>(ends + (int64_t)r0 * m);
        const int ne = (rows_here * m + 3) >> 2;
        for (int i = threadIdx.x; i < ne; i += ROWS) reinterpret_cast<int4 *>(se)[i] = ld_stream(ge + i);
        for (int i = threadIdx.x; i < m; i += ROWS) st[i] = table[i];
    }
    __syncthreads();
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
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_LOOP:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra DONE;\n\t"
        "bra WAIT_LOOP;\n"
        "DONE:\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

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

// =============================================================================
// Pattern format (inc/compress.hpp:48-76; spmv: inc/kernels.hpp:25,35-36;
// PAPER.md:797-813 List 1).
// =============================================================================
struct PatternArgs {
    const int32_t *ids;        // row_pattern, local row 0
    const double *x;
    double *y;
    int64_t g0;                // x index of the diagonal of local row 0: row_offset - x_col0
    int64_t x_len;
    const int32_t *disp_off;   // n_patterns + 1
    const int32_t *disp;       // displacements
    const int32_t *ends;       // n_patterns * m
    const double *table;       // m
    const uint32_t *masks;     // n_patterns (box plan)
    int n_patterns, m, disp_total;
    int row_begin, row_end;
    // box plan
    int sy, plane_lines;       // sy = stride of dy; plane_lines = sz / sy
    double v_off, v_center;
    int prefetch;              // L2 prefetch distance in lines
    int prefetch_l1;           // L1 prefetch distance in lines (v3), 0 = off
    int debug_nochain;         // measurement only: skip the FP64 chains (y = centre operand)
};

// List 1, one row: groups in table order, per element value * x.
__device__ __forceinline__ double pattern_row(const PatternArgs &p, const int32_t *disp, const int32_t *ends,
                                              const double *table, int id, int64_t xi) {
    double acc = 0.0;
    int idx = 0;
    const int32_t *d = disp + p.disp_off[id];
    const int32_t *e = ends + id * p.m;
    for (int k = 0; k < p.m; k++) {
        const double a_ij = table[k];
        const int end = e[k];
        for (; idx < end; idx++) acc = __dadd_rn(acc, __dmul_rn(a_ij, __ldg(p.x + (xi + d[idx]))));
    }
    return acc;
}

__device__ __noinline__ double pattern_row_cold(const PatternArgs &p, int id, int64_t xi) {
    return pattern_row(p, p.disp, p.ends, p.table, id, xi);
}

// Generic kernel: thread per row, any dictionary.  DICT_SMEM keeps the dictionary
// (displacements, ends, table, offsets) in shared memory when it is small.
constexpr int kDictSmemDisp = 2048;  // displacements
constexpr int kDictSmemPat = 64;     // patterns
constexpr int kDictSmemTab = 8;      // table entries

template <bool DICT_SMEM>
__global__ void __launch_bounds__(256) spmv_pattern_generic_kernel(PatternArgs p) {
    __shared__ int32_t s_disp[DICT_SMEM ? kDictSmemDisp : 1];
    __shared__ int32_t s_ends[DICT_SMEM ? kDictSmemPat * kDictSmemTab : 1];
    __shared__ int32_t s_off[DICT_SMEM ? kDictSmemPat + 1 : 1];
    __shared__ double s_tab[DICT_SMEM ? kDictSmemTab : 1];
    PatternArgs q = p;
    if (DICT_SMEM) {
        for (int i = threadIdx.x; i < p.disp_total; i += blockDim.x) s_disp[i] = p.disp[i];
        for (int i = threadIdx.x; i < p.n_patterns * p.m; i += blockDim.x) s_ends[i] = p.ends[i];
        for (int i = threadIdx.x; i <= p.n_patterns; i += blockDim.x) s_off[i] = p.disp_off[i];
        for (int i = threadIdx.x; i < p.m; i += blockDim.x) s_tab[i] = p.table[i];
        __syncthreads();
        q.disp_off = s_off;
    }
    const int r = p.row_begin + blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.row_end) return;
    const int id = ld_stream(p.ids + r);
    if (id < 0) return;  // exception row: written by the exception kernel
    p.y[r] = pattern_row(q, DICT_SMEM ? s_disp : p.disp, DICT_SMEM ? s_ends : p.ends,
                         DICT_SMEM ? s_tab : p.table, id, p.g0 + r);
}

// -----------------------------------------------------------------------------
// Sliding-window ("box") kernel.  Applies when the dictionary's dominant pattern
// is the 3x3x3 box {dx + sy*dy + sz*dz} (BoxPlan); every other pattern that is a
// subset of it is a 27-bit mask, anything else falls back per lane to List 1.
//
// Rows of the range are indexed r = a + sy*(b + plane_lines*c).  A warp owns 32
// consecutive a at one c and marches b; a thread keeps the x values of lines
// b-1, b, b+1 (+ one line of look-ahead) x {dz} x {dx} in registers, so each new
// row costs 9 coalesced loads instead of 27, all of them L1/L2 hits after the
// first touch.  The warps of a CTA sit on consecutive c (z planes) and share the
// lines through L1.  The per-row work is still driven by the streamed pattern id:
// id -> mask -> predicated accumulation in the dictionary's (value, displacement)
// order, i.e. exactly the reference's summation order.
// -----------------------------------------------------------------------------
template <bool GUARD>
__device__ __forceinline__ double box_load(const double *__restrict__ x, int64_t idx, int64_t x_len) {
    if (GUARD) {
        if ((uint64_t)idx >= (uint64_t)x_len) return 0.0;
    }
    return __ldg(x + idx);
}

constexpr uint32_t kFullBox = 0x07FFFFFFu;

// One warp: 32 consecutive a, Q consecutive planes c0..c0+Q-1 per thread (Q
// independent accumulation chains), marching nb lines.  Window w[slot][plane][dx]
// holds lines j-1, j, j+1 (+LA lines of look-ahead) of planes c0-1..c0+Q.
template <int Q, int LA, bool OFF_NEG1, int CENTER_POS, bool GUARD>
__device__ __forceinline__ void box_march(const PatternArgs &p, const uint32_t *s_masks, int64_t r, int nb,
                                          int64_t n_rows, int nq, bool lane_ok, bool pf_lo, bool pf_hi) {
    constexpr int S = 3 + LA;
    constexpr int P = Q + 2;
    const int64_t sy = p.sy;
    const int64_t sz = sy * p.plane_lines;
    const double *__restrict__ x = p.x;
    const int32_t *__restrict__ ids = p.ids + p.row_begin;
    double *__restrict__ y = p.y + p.row_begin;
    int64_t xi = p.g0 + p.row_begin + r;  // x index of the diagonal of (current line, plane c0)
    double w[S][P][3];
    auto load_line = [&](int slot, int64_t centre) {
#pragma unroll
        for (int pz = 0; pz < P; pz++)
#pragma unroll
            for (int dx = 0; dx < 3; dx++)
                w[slot][pz][dx] = box_load<GUARD>(x, centre + (pz - 1) * sz + (dx - 1), p.x_len);
    };
    load_line(S - 1, xi - sy);
    load_line(0, xi);
    if (LA) load_line(1, xi + sy);
    int id_next[Q];
#pragma unroll
    for (int q = 0; q < Q; q++)
        id_next[q] = (lane_ok && q < nq && r + q * sz < n_rows) ? ld_stream(ids + r + q * sz) : -1;
    const int pf = p.prefetch;
    const double vc = p.v_center, vo = p.v_off;
#pragma unroll 1
    for (int j0 = 0; j0 < nb; j0 += S) {
#pragma unroll
        for (int k = 0; k < S; k++) {
            const int j = j0 + k;
            if (j < nb) {
                load_line((k + 1 + LA) % S, xi + (1 + LA) * sy);
                int id[Q];
                uint32_t mk[Q];
                bool full = true;
#pragma unroll
                for (int q = 0; q < Q; q++) {
                    id[q] = id_next[q];
                    id_next[q] = (lane_ok && q < nq && j + 1 < nb && r + sy + q * sz < n_rows)
                                     ? ld_stream(ids + r + sy + q * sz) : -1;
                    mk[q] = id[q] >= 0 ? (s_masks ? s_masks[id[q]] : __ldg(p.masks + id[q])) : 0u;
                    full = full && (mk[q] == kFullBox);
                }
                if (pf > 0) {  // pull the lines `pf` steps ahead from HBM into L2
                    const int64_t t = xi + (int64_t)pf * sy;
#pragma unroll
                    for (int q = 0; q < Q; q++) {
                        const int64_t tq = t + q * sz;
                        if ((uint64_t)tq < (uint64_t)p.x_len) prefetch_l2(x + tq);
                        const int64_t rq = r + (int64_t)pf * sy + q * sz;
                        if (q < nq && rq < n_rows) prefetch_l2(ids + rq);
                    }
                    if (pf_lo && (uint64_t)(t - sz) < (uint64_t)p.x_len) prefetch_l2(x + t - sz);
                    if (pf_hi && (uint64_t)(t + Q * sz) < (uint64_t)p.x_len) prefetch_l2(x + t + Q * sz);
                }
                double acc[Q];
#pragma unroll
                for (int q = 0; q < Q; q++) acc[q] = 0.0;
                const int sl[3] = {(k + S - 1) % S, k, (k + 1) % S};
                if (__all_sync(0xffffffffu, full)) {
                    // every row of this step has the full box: no selects on the chain
                    if (CENTER_POS == 0) {
#pragma unroll
                        for (int q = 0; q < Q; q++) acc[q] = __dadd_rn(acc[q], __dmul_rn(vc, w[sl[1]][q + 1][1]));
                    }
#pragma unroll
                    for (int t = 0; t < 27; t++) {
                        if (t == 13 && CENTER_POS != 2) continue;
                        const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            const double e = w[sl[dy]][q + dz][dx];
                            acc[q] = OFF_NEG1 ? __dsub_rn(acc[q], e) : __dadd_rn(acc[q], __dmul_rn(vo, e));
                        }
                    }
                    if (CENTER_POS == 1) {
#pragma unroll
                        for (int q = 0; q < Q; q++) acc[q] = __dadd_rn(acc[q], __dmul_rn(vc, w[sl[1]][q + 1][1]));
                    }
                } else {
                    // Masked rows: an absent entry contributes +0.0.  acc starts at +0.0 and can
                    // never become -0.0 (round to nearest), so adding +-0.0 leaves it unchanged
                    // bit for bit: identical to skipping the term as the reference does.
                    if (CENTER_POS == 0) {
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            const double pr = __dmul_rn(vc, w[sl[1]][q + 1][1]);
                            acc[q] = __dadd_rn(acc[q], (mk[q] >> 13 & 1u) ? pr : 0.0);
                        }
                    }
#pragma unroll
                    for (int t = 0; t < 27; t++) {
                        if (t == 13 && CENTER_POS != 2) continue;
                        const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            const double e = w[sl[dy]][q + dz][dx];
                            const bool on = mk[q] >> t & 1u;
                            if (OFF_NEG1) acc[q] = __dsub_rn(acc[q], on ? e : 0.0);
                            else acc[q] = __dadd_rn(acc[q], on ? __dmul_rn(vo, e) : 0.0);
                        }
                    }
                    if (CENTER_POS == 1) {
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            const double pr = __dmul_rn(vc, w[sl[1]][q + 1][1]);
                            acc[q] = __dadd_rn(acc[q], (mk[q] >> 13 & 1u) ? pr : 0.0);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < Q; q++)  // patterns outside the box: List 1 per lane
                        if (mk[q] == kGenericMask) acc[q] = pattern_row(p, p.disp, p.ends, p.table, id[q], xi + q * sz);
                }
#pragma unroll
                for (int q = 0; q < Q; q++)
                    if (id[q] >= 0) y[r + q * sz] = acc[q];
                r += sy;
                xi += sy;
            }
        }
    }
}

template <int R, int WC, int Q, int LA, bool OFF_NEG1, int CENTER_POS>
__global__ void __launch_bounds__(WC * 32) spmv_pattern_box_kernel(PatternArgs p, int n_planes) {
    __shared__ uint32_t s_masks_buf[kDictSmemPat];
    const uint32_t *s_masks = nullptr;
    if (p.n_patterns <= kDictSmemPat) {
        for (int i = threadIdx.x; i < p.n_patterns; i += WC * 32) s_masks_buf[i] = p.masks[i];
        __syncthreads();
        s_masks = s_masks_buf;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int a = blockIdx.x * 32 + lane;
    const int c0 = (blockIdx.z * WC + warp) * Q;
    const int b0 = blockIdx.y * R;
    if (c0 >= n_planes) return;  // warp-uniform
    const int nb = min(R, p.plane_lines - b0);
    const int nq = min(Q, n_planes - c0);
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sy = p.sy, sz = sy * p.plane_lines;
    const int64_t r = a + sy * (b0 + (int64_t)p.plane_lines * c0);
    const int64_t r_warp = r - lane;
    if (r_warp >= n_rows) return;  // warp-uniform
    const bool lane_ok = a < p.sy;
    // Guard-free marching when every speculative window load of this warp is in range.
    const int64_t xi0 = p.g0 + p.row_begin + r_warp;
    const int64_t lo = xi0 - sy - sz - 1;
    const int64_t hi = xi0 + 31 + (int64_t)(nb + 1 + LA) * sy + (int64_t)Q * sz + 1;
    const bool safe = lo >= 0 && hi < p.x_len;
    const bool pf_lo = warp == 0, pf_hi = (warp == WC - 1) || (c0 + Q >= n_planes);
    if (safe) box_march<Q, LA, OFF_NEG1, CENTER_POS, false>(p, s_masks, r, nb, n_rows, nq, lane_ok, pf_lo, pf_hi);
    else box_march<Q, LA, OFF_NEG1, CENTER_POS, true>(p, s_masks, r, nb, n_rows, nq, lane_ok, pf_lo, pf_hi);
}

// -----------------------------------------------------------------------------
// Sliding-window kernel, version 3 ("box3"): the same plan as above with two
// adjacent columns, Q planes and LPS lines per thread and step.
//   * x-tiling: a thread owns columns a0, a0+1, so one 128-bit load brings both of
//     its own elements of a line and two 64-bit loads bring the halo columns
//     a0-1 / a0+2: 3 loads per (line, plane) serve 2 rows (v2: 3 loads per row).
//   * 2*Q*LPS independent accumulation chains per thread: the reference's fixed
//     summation order makes every row a 27-deep dependent DADD chain, so the FP64
//     pipe is only kept busy by many chains in flight per scheduler.
//   * All addresses are a warp-uniform base pointer (bumped once per step) plus a
//     per-thread 32-bit offset.
//   * Row masks: rows whose only missing entries are the nine dx=-1 (or dx=+1)
//     ones -- the x-boundary rows, which sit in the thread's edge column -- are
//     served by zeroing those nine halo operands; any other partial mask takes the
//     fully masked chain.  Absent operands are +0.0, which leaves the accumulator
//     unchanged bit for bit (it can never be -0.0), i.e. the reference's order.
// Interior tiles (every window load and prefetch in range) march guard-free; edge
// tiles use the guarded v2 march.  Needs even strides/offsets and 16-byte aligned
// x, y, ids; otherwise the v2 kernel above is used.
// -----------------------------------------------------------------------------
constexpr uint32_t kLBits = 0x1249249u;  // box entries with dx = -1
constexpr uint32_t kRBits = 0x4924924u;  // box entries with dx = +1

template <int Q, int S, int LPS, bool OFF_NEG1, int CENTER_POS, int MODE, bool SELL, bool SELR>
__device__ __forceinline__ void box3_chain(const double (&w)[S][Q + 2][4], int kb, const uint32_t (&mk)[LPS][Q][2],
                                           const bool (&zl)[LPS][Q], const bool (&zr)[LPS][Q], double vc, double vo,
                                           double (&acc)[LPS][Q][2]) {
    // MODE 0: operands straight from the window (with SELL/SELR: halo operands zeroed per lane)
    // MODE 1: every operand selected by its mask bit
    // line l of the step reads slots (kb+l-1, kb+l, kb+l+1) mod S for dy = -1, 0, +1
    double hl[LPS][Q][3][3], hr[LPS][Q][3][3];
    if (MODE == 0 && (SELL || SELR)) {
#pragma unroll
        for (int l = 0; l < LPS; l++)
#pragma unroll
            for (int q = 0; q < Q; q++)
#pragma unroll
                for (int dz = 0; dz < 3; dz++)
#pragma unroll
                    for (int dy = 0; dy < 3; dy++) {
                        const int s = (kb + l + dy + S - 1) % S;
                        if (SELL) hl[l][q][dz][dy] = zl[l][q] ? 0.0 : w[s][q + dz][0];
                        if (SELR) hr[l][q][dz][dy] = zr[l][q] ? 0.0 : w[s][q + dz][3];
                    }
    }
#pragma unroll
    for (int l = 0; l < LPS; l++)
#pragma unroll
        for (int q = 0; q < Q; q++) acc[l][q][0] = acc[l][q][1] = 0.0;
    auto centre = [&]() {
#pragma unroll
        for (int l = 0; l < LPS; l++)
#pragma unroll
            for (int q = 0; q < Q; q++)
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    const double pr = __dmul_rn(vc, w[(kb + l) % S][q + 1][i + 1]);
                    acc[l][q][i] = __dadd_rn(acc[l][q][i], (MODE == 1 && !(mk[l][q][i] >> 13 & 1u)) ? 0.0 : pr);
                }
    };
    if (CENTER_POS == 0) centre();
#pragma unroll
    for (int t = 0; t < 27; t++) {
        if (t == 13 && CENTER_POS != 2) continue;
        const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
#pragma unroll
        for (int l = 0; l < LPS; l++)
#pragma unroll
            for (int q = 0; q < Q; q++)
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    double e = w[(kb + l + dy + S - 1) % S][q + dz][i + dx];
                    if (MODE == 0 && SELL && i + dx == 0) e = hl[l][q][dz][dy];
                    if (MODE == 0 && SELR && i + dx == 3) e = hr[l][q][dz][dy];
                    if (OFF_NEG1) {
                        if (MODE == 1) e = (mk[l][q][i] >> t & 1u) ? e : 0.0;
                        acc[l][q][i] = __dsub_rn(acc[l][q][i], e);
                    } else {
                        double pr = __dmul_rn(vo, e);
                        if (MODE == 1) pr = (mk[l][q][i] >> t & 1u) ? pr : 0.0;
                        acc[l][q][i] = __dadd_rn(acc[l][q][i], pr);
                    }
                }
    }
    if (CENTER_POS == 1) centre();
}

// Row classes (shared-memory tables indexed by pattern id + 1; entry 0 serves exception
// rows, id = -1, which are computed as full rows and never stored).  cls0 is for rows in
// the thread's left column, cls1 for its right column:
//   0 full box; 1 (cls0) only the nine dx=-1 entries missing; 2 (cls1) only the nine
//   dx=+1 entries missing; 4 any other mask (fully masked chain / List 1).
struct Box3Smem {
    uint32_t cls0, cls1, masks;  // 32-bit shared addresses of the three tables
};

template <int Q, int LPS, bool OFF_NEG1, int CENTER_POS>
__device__ __forceinline__ void box3_march(const PatternArgs &p, const Box3Smem sm, const double *__restrict__ xw,
                                           const int32_t *__restrict__ idw, double *__restrict__ yw, int64_t xi_w, int lane,
                                           int nb, bool lane_ok, int nq) {
    constexpr int S = LPS + 2, P = Q + 2;
    constexpr int U = (S % LPS == 0) ? S / LPS : S;  // steps until the slot pattern repeats
    const int sy = p.sy;
    const int sz = sy * p.plane_lines;
    const int lo = lane * 2;
    constexpr int dbg = 0;  // ablation switches of profiles/r01_ablation_*.log (1 no chain, 2 no halo loads, 4 no ids, 8 no prefetch)
    double w[S][P][4];
    auto load_line = [&](int slot, int line_off) {
#pragma unroll
        for (int pz = 0; pz < P; pz++) {
            const double *pl = xw + (lo + (pz - 1) * sz + line_off);
            const double2 v = __ldg(reinterpret_cast<const double2 *>(pl));
            if (dbg & 2) {  // measurement only: no halo loads
                w[slot][pz][0] = v.y;
                w[slot][pz][3] = v.x;
            } else {
                w[slot][pz][0] = __ldg(pl - 1);
                w[slot][pz][3] = __ldg(pl + 2);
            }
            w[slot][pz][1] = v.x;
            w[slot][pz][2] = v.y;
        }
    };
    bool vq[Q];  // rows of plane q exist for this lane
#pragma unroll
    for (int q = 0; q < Q; q++) vq[q] = lane_ok && q < nq;
    auto load_ids = [&](int q, bool line_ok, int line_off) {
        int2 r = make_int2(-1, -1);  // rows outside the tile's valid columns / planes / lines: computed, never stored
        if (dbg & 4) r = make_int2(13, 13);  // measurement only: no id stream
        else if (vq[q] && line_ok) {
            const int2 *ptr = reinterpret_cast<const int2 *>(idw + (lo + q * sz + line_off));
            asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(ptr));
        }
        return r;
    };
    load_line(S - 1, -sy);
    load_line(0, 0);
    int2 idn[LPS][Q];
#pragma unroll
    for (int l = 0; l < LPS; l++)
#pragma unroll
        for (int q = 0; q < Q; q++) idn[l][q] = load_ids(q, l < nb, l * sy);
    const int pf = p.prefetch * LPS * sy;  // L2 prefetch distance in elements
    const double vc = p.v_center, vo = p.v_off;
#pragma unroll 1
    for (int j0 = 0; j0 < nb; j0 += U * LPS) {
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int jb = j0 + u * LPS;   // first line of this step
            const int kb = (u * LPS) % S;  // its slot
            if (jb < nb) {
#pragma unroll
                for (int l = 0; l < LPS; l++) load_line((kb + 1 + l) % S, (1 + l) * sy);
                int id[LPS][Q][2];
                uint32_t c0[LPS][Q], c1[LPS][Q], wv = 0;
#pragma unroll
                for (int l = 0; l < LPS; l++)
#pragma unroll
                    for (int q = 0; q < Q; q++) {
                        id[l][q][0] = idn[l][q].x;
                        id[l][q][1] = idn[l][q].y;
                        idn[l][q] = load_ids(q, jb + LPS + l < nb, (LPS + l) * sy);
                        c0[l][q] = lds_u32(sm.cls0 + 4 + 4 * id[l][q][0]);
                        c1[l][q] = lds_u32(sm.cls1 + 4 + 4 * id[l][q][1]);
                        wv |= c0[l][q] | c1[l][q];
                    }
                if (pf > 0 && !(dbg & 8)) {  // pull the lines `prefetch` steps ahead from HBM into L2
                    // (one TMA bulk prefetch per segment, cp.async.bulk.prefetch.L2, measured identical:
                    //  profiles/r01_ablation_bulk_l2_prefetch.log; it also needs 16-byte aligned id rows)
#pragma unroll
                    for (int l = 0; l < LPS; l++)
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            prefetch_l2(xw + (lo + q * sz + l * sy + pf));
                            prefetch_l2(idw + (lo + q * sz + l * sy + pf));
                        }
                }
                double acc[LPS][Q][2];
                uint32_t mk[LPS][Q][2];
                bool zl[LPS][Q], zr[LPS][Q];
                const unsigned vote = __reduce_or_sync(0xffffffffu, wv);  // 1 some L-partial, 2 some R-partial, 4 other
                if (dbg & 1) {
#pragma unroll
                    for (int l = 0; l < LPS; l++)
#pragma unroll
                        for (int q = 0; q < Q; q++)
#pragma unroll
                            for (int i = 0; i < 2; i++) acc[l][q][i] = w[(kb + l) % S][q + 1][i + 1] + w[(kb + l + 1) % S][q + 2][i + 2];
                } else if (vote == 0) {
                    box3_chain<Q, S, LPS, OFF_NEG1, CENTER_POS, 0, false, false>(w, kb, mk, zl, zr, vc, vo, acc);
                } else if (vote == 1 || vote == 2) {
#pragma unroll
                    for (int l = 0; l < LPS; l++)
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            zl[l][q] = c0[l][q] != 0;
                            zr[l][q] = c1[l][q] != 0;
                        }
                    if (vote == 1) box3_chain<Q, S, LPS, OFF_NEG1, CENTER_POS, 0, true, false>(w, kb, mk, zl, zr, vc, vo, acc);
                    else box3_chain<Q, S, LPS, OFF_NEG1, CENTER_POS, 0, false, true>(w, kb, mk, zl, zr, vc, vo, acc);
                } else {
#pragma unroll
                    for (int l = 0; l < LPS; l++)
#pragma unroll
                        for (int q = 0; q < Q; q++)
#pragma unroll
                            for (int i = 0; i < 2; i++) mk[l][q][i] = lds_u32(sm.masks + 4 + 4 * id[l][q][i]);
                    box3_chain<Q, S, LPS, OFF_NEG1, CENTER_POS, 1, false, false>(w, kb, mk, zl, zr, vc, vo, acc);
#pragma unroll
                    for (int l = 0; l < LPS; l++)
#pragma unroll
                        for (int q = 0; q < Q; q++)
#pragma unroll
                            for (int i = 0; i < 2; i++)  // patterns outside the box: List 1 per lane
                                if (mk[l][q][i] == kGenericMask)
                                    acc[l][q][i] = pattern_row(p, p.disp, p.ends, p.table, id[l][q][i],
                                                               xi_w + lo + (int64_t)l * sy + q * (int64_t)sz + i);
                }
#pragma unroll
                for (int l = 0; l < LPS; l++)
#pragma unroll
                    for (int q = 0; q < Q; q++) {
                        double *dst = yw + (lo + q * sz + l * sy);
                        if ((id[l][q][0] | id[l][q][1]) >= 0)
                            *reinterpret_cast<double2 *>(dst) = make_double2(acc[l][q][0], acc[l][q][1]);
                        else {
                            if (id[l][q][0] >= 0) dst[0] = acc[l][q][0];
                            if (id[l][q][1] >= 0) dst[1] = acc[l][q][1];
                        }
                    }
                xw += LPS * sy;
                idw += LPS * sy;
                yw += LPS * sy;
                xi_w += (int64_t)LPS * sy;
            }
        }
    }
}

// Fills the class / mask tables of Box3Smem (entry 0 = exception rows -> full box).
__device__ __forceinline__ void box3_fill_tables(const PatternArgs &p, uint32_t *cls0, uint32_t *cls1, uint32_t *masks,
                                                 int tid, int nthreads) {
    for (int i = tid; i <= p.n_patterns; i += nthreads) {
        const uint32_t m = i == 0 ? kFullBox : p.masks[i - 1];
        masks[i] = m;
        cls0[i] = m == kFullBox ? 0u : (m == (kFullBox & ~kLBits) ? 1u : 4u);
        cls1[i] = m == kFullBox ? 0u : (m == (kFullBox & ~kRBits) ? 2u : 4u);
    }
}

// grid edges / slab ends / ragged ranges: the guarded one-column march of the v2 kernel, per half warp-tile
template <int Q, bool OFF_NEG1, int CENTER_POS>
__device__ __noinline__ void box3_edge_tile(const PatternArgs &p, const uint32_t *s_masks, int64_t r_w, int lane, int nb,
                                            int64_t n_rows, int nq, int cols_ok) {
#pragma unroll 1
    for (int half = 0; half < 2; half++)
        box_march<Q, 0, OFF_NEG1, CENTER_POS, true>(p, s_masks, r_w + half * 32 + lane, nb, n_rows, nq,
                                                    half * 32 + lane < cols_ok, false, false);
}

template <int R, int WC, int Q, int LPS, int MINB, bool OFF_NEG1, int CENTER_POS, int WA = 1>
__global__ void __launch_bounds__(WC * 32, MINB) spmv_pattern_box3_kernel(PatternArgs p, int n_planes) {
    __shared__ uint32_t s_cls0[kDictSmemPat + 1], s_cls1[kDictSmemPat + 1], s_masks1[kDictSmemPat + 1];
    box3_fill_tables(p, s_cls0, s_cls1, s_masks1, threadIdx.x, WC * 32);
    const uint32_t *s_masks = s_masks1 + 1;
    __syncthreads();
    Box3Smem sm;
    sm.cls0 = (uint32_t)__cvta_generic_to_shared(s_cls0);
    sm.cls1 = (uint32_t)__cvta_generic_to_shared(s_cls1);
    sm.masks = (uint32_t)__cvta_generic_to_shared(s_masks1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // WA warps of the CTA sit side by side along x (a CTA then reads contiguous runs of WA*512 bytes
    // per line and plane), the remaining WC/WA along z.
    const int a_w = (blockIdx.x * WA + warp % WA) * 64;  // first column of the warp
    const int c0 = (blockIdx.z * (WC / WA) + warp / WA) * Q;
    const int b0 = blockIdx.y * R;
    if (c0 >= n_planes) return;
    const int nb = min(R, p.plane_lines - b0);
    const int nq = min(Q, n_planes - c0);
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sy = p.sy, sz = sy * p.plane_lines;
    const int64_t r_w = a_w + sy * (b0 + (int64_t)p.plane_lines * c0);  // relative row of (lane 0, first line, plane c0)
    if (r_w >= n_rows) return;
    const int cols_ok = min(64, p.sy - a_w);
    const int64_t xi_w = p.g0 + p.row_begin + r_w;
    const int pf = (p.prefetch > 0 ? p.prefetch : 0) * LPS;
    // Guard-free march when every row of the tile's valid columns/planes/lines is in the row range
    // and every window load and prefetch of the warp is in range; rows of missing columns / planes
    // / lines are computed on in-range data and dropped.
    const int nb_up = (nb + LPS - 1) / LPS * LPS;
    const int64_t last_row = r_w + (cols_ok - 1) + (int64_t)(nb - 1) * sy + (int64_t)(nq - 1) * sz;
    const int64_t x_lo = xi_w - sy - sz - 1;
    const int64_t x_hi = xi_w + 64 + (int64_t)(nb_up + LPS + pf) * sy + (int64_t)Q * sz + 1;
    const int64_t id_hi = r_w + 64 + (int64_t)(nb_up + LPS + pf) * sy + (int64_t)(nq - 1) * sz;  // ids prefetch reach
    const bool interior = last_row < n_rows && x_lo >= 0 && x_hi < p.x_len && id_hi <= n_rows + 1024;
    if (interior) {
        box3_march<Q, LPS, OFF_NEG1, CENTER_POS>(p, sm, p.x + xi_w, p.ids + p.row_begin + r_w, p.y + p.row_begin + r_w, xi_w,
                                                 lane, nb, lane * 2 + 1 < cols_ok, nq);
    } else {
        box3_edge_tile<Q, OFF_NEG1, CENTER_POS>(p, s_masks, r_w, lane, nb, n_rows, nq, cols_ok);
    }
}

// -----------------------------------------------------------------------------
// Sliding-window kernel, version 4 ("box5"): box3's arithmetic fed from a
// multi-stage shared-memory ring.  The stall profile of box3 showed the FP64 chains
// were not the limit: every step exposed L2/HBM latency on its serial setup (window
// loads, ids -> mask -> vote -> branch) with only ~2.5 warps per scheduler.  Here the
// CTA's x lines (WC*Q+2 planes x 68 doubles) and pattern ids (WC*Q planes x 64 ints)
// of line l are copied global -> shared with cp.async (16-byte chunks, L2 only) DEPTH
// lines ahead of their use, so the per-step critical path only sees shared-memory
// latency, and the z halo between the warps of a CTA is fetched once per CTA.
// Interior CTAs only (all copies in range); edge CTAs use the guarded v2 march.
// Needs strides and offsets that are multiples of 4 rows and 16-byte aligned arrays.
// -----------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_smem), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int R, int WC, int Q, int DEPTH, int MINB, bool OFF_NEG1, int CENTER_POS>
__global__ void __launch_bounds__(WC * 32, MINB) spmv_pattern_box5_kernel(PatternArgs p, int n_planes) {
    constexpr int T = WC * 32;
    constexpr int NP = WC * Q;         // planes computed by the CTA
    constexpr int XP = NP + 2;         // x planes staged (one halo plane each side)
    constexpr int XW = 68;             // staged doubles per x line: columns a_w-2 .. a_w+65
    constexpr int XCH = XP * (XW / 2); // 16-byte chunks of x per stage
    constexpr int ICH = NP * 16;       // 16-byte chunks of ids per stage
    constexpr int NCH = XCH + ICH;
    constexpr int PER = (NCH + T - 1) / T;
    constexpr int S = 3, P = Q + 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *xs = reinterpret_cast<double *>(smem_raw);                              // [DEPTH][XP][XW]
    int32_t *is = reinterpret_cast<int32_t *>(smem_raw + (size_t)DEPTH * XP * XW * 8);  // [DEPTH][NP][64]
    __shared__ uint32_t s_masks[kDictSmemPat];
    for (int i = threadIdx.x; i < p.n_patterns; i += T) s_masks[i] = p.masks[i];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int a_w = blockIdx.x * 64;
    const int c0 = blockIdx.z * NP;   // first plane of the CTA
    const int b0 = blockIdx.y * R;
    const int nb = min(R, p.plane_lines - b0);
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sy64 = p.sy, sz64 = sy64 * p.plane_lines;
    const int64_t r_c = a_w + sy64 * (b0 + (int64_t)p.plane_lines * c0);  // relative row of (column a_w, line b0, plane c0)
    const int cols_ok = min(64, p.sy - a_w);
    const int nq_cta = min(NP, n_planes - c0);
    const int64_t xi_c = p.g0 + p.row_begin + r_c;
    // interior CTA: every staged byte (lines -1..nb, planes c0-1..c0+NP) is inside x, every id read inside ids
    const int64_t x_lo = xi_c - sy64 - sz64 - 2;
    const int64_t x_hi = xi_c + 66 + (int64_t)nb * sy64 + (int64_t)NP * sz64;
    const int64_t last_row = r_c + (cols_ok - 1) + (int64_t)(nb - 1) * sy64 + (int64_t)(nq_cta - 1) * sz64;
    const bool interior = x_lo >= 0 && x_hi < p.x_len && last_row < n_rows && cols_ok == 64;
    __syncthreads();
    if (!interior) {  // CTA-uniform: grid edges, slab ends, ragged ranges
        const int cw = c0 + warp * Q;
        if (cw < n_planes && r_c + (int64_t)warp * Q * sz64 < n_rows)
            box3_edge_tile<Q, OFF_NEG1, CENTER_POS>(p, s_masks, r_c + (int64_t)warp * Q * sz64, lane, nb, n_rows,
                                                    min(Q, n_planes - cw), cols_ok);
        return;
    }
    const int sy = p.sy, sz = sy * p.plane_lines;
    // ---- per-thread copy plan: chunk c = tid + k*T -> (source offset, shared offset)
    const double *xg = p.x + xi_c;                       // (column a_w, line b0, plane c0)
    const int32_t *ig = p.ids + p.row_begin + r_c;
    int src_off[PER];       // elements, relative to xg (doubles) or ig (ints), for line 0
    uint32_t dst_off[PER];  // bytes from the start of a stage's x (or ids) area
    int kind[PER];          // 0 x, 1 ids, 2 none
    const uint32_t xs_base = (uint32_t)__cvta_generic_to_shared(xs);
    const uint32_t is_base = (uint32_t)__cvta_generic_to_shared(is);
#pragma unroll
    for (int k = 0; k < PER; k++) {
        const int c = threadIdx.x + k * T;
        if (c < XCH) {
            const int pz = c / (XW / 2), j = c % (XW / 2);
            kind[k] = 0;
            src_off[k] = (pz - 1) * sz - 2 + 2 * j;
            dst_off[k] = (uint32_t)((pz * XW + 2 * j) * 8);
        } else if (c < NCH) {
            const int q = (c - XCH) / 16, j = (c - XCH) % 16;
            kind[k] = q < nq_cta ? 1 : 2;
            src_off[k] = q * sz + 4 * j;
            dst_off[k] = (uint32_t)((q * 64 + 4 * j) * 4);
        } else {
            kind[k] = 2; src_off[k] = 0; dst_off[k] = 0;
        }
    }
    auto fetch = [&](int line) {  // stage line `line` (-1 .. nb) into ring slot (line+1) % DEPTH; always one group
        if (line <= nb) {
            const int slot = (line + 1) % DEPTH;
#pragma unroll
            for (int k = 0; k < PER; k++) {
                if (kind[k] == 0)
                    cp_async16(xs_base + (uint32_t)(slot * XP * XW * 8) + dst_off[k], xg + (src_off[k] + line * sy));
                else if (kind[k] == 1 && line >= 0 && line < nb)
                    cp_async16(is_base + (uint32_t)(slot * NP * 64 * 4) + dst_off[k], ig + (src_off[k] + line * sy));
            }
        }
        cp_async_commit();
    };
    // ---- consumer view: this warp's planes are staged x planes warp*Q .. warp*Q+Q+1
    const int pw = warp * Q;
    const bool warp_on = c0 + pw < n_planes;
    const int nq = min(Q, n_planes - (c0 + pw));
    double w[S][P][4];
    auto load_line = [&](int wslot, int line) {
        const double *base = xs + ((line + 1) % DEPTH) * (XP * XW) + pw * XW + 2 * lane;
#pragma unroll
        for (int pz = 0; pz < P; pz++) {
            const double *pl = base + pz * XW;
            const double2 v = *reinterpret_cast<const double2 *>(pl + 2);
            w[wslot][pz][0] = pl[1];
            w[wslot][pz][1] = v.x;
            w[wslot][pz][2] = v.y;
            w[wslot][pz][3] = pl[4];
        }
    };
#pragma unroll
    for (int l = -1; l < DEPTH - 1; l++) fetch(l);  // DEPTH groups in flight: lines -1 .. DEPTH-2
    cp_async_wait<DEPTH - 2>();                     // lines -1 and 0 have landed
    __syncthreads();
    load_line(S - 1, -1);
    load_line(0, 0);
    double *yw = p.y + p.row_begin + r_c + (int64_t)pw * sz64 + 2 * lane;
    const double vc = p.v_center, vo = p.v_off;
    // L2 prefetch only while its farthest address stays inside x and ids
    const int pf = (x_hi + (int64_t)(DEPTH + p.prefetch) * sy64 < p.x_len &&
                    last_row + (int64_t)(DEPTH + p.prefetch) * sy64 < n_rows) ? p.prefetch : 0;
#pragma unroll 1
    for (int j0 = 0; j0 < nb; j0 += S) {
#pragma unroll
        for (int k = 0; k < S; k++) {
            const int j = j0 + k;
            if (j < nb) {  // CTA-uniform
                cp_async_wait<DEPTH - 3>();  // line j+1 has landed (groups up to line j+DEPTH-2 are committed)
                __syncthreads();             // ... for every thread's copies; slot of line j-1 is free again
                fetch(j + DEPTH - 1);
                if (pf > 0 && lane < 8) {    // a little further ahead: HBM -> L2, one request per 128-byte line
                    const int line = j + DEPTH - 1 + pf;
#pragma unroll
                    for (int q = 0; q < Q; q++) {
                        prefetch_l2(xg + ((pw + q) * sz + line * sy + 16 * lane));
                        if (lane < 2) prefetch_l2(ig + ((pw + q) * sz + line * sy + 32 * lane));
                    }
                    if (warp == 0) prefetch_l2(xg + (-sz + line * sy + 16 * lane));
                    if (warp == WC - 1) prefetch_l2(xg + (NP * sz + line * sy + 16 * lane));
                }
                load_line((k + 1) % S, j + 1);
                if (warp_on) {
                    int id[1][Q][2];
                    uint32_t mk[1][Q][2];
                    bool zl[1][Q], zr[1][Q], other = false, anyl = false, anyr = false;
                    const int32_t *idl = is + ((j + 1) % DEPTH) * (NP * 64) + pw * 64 + 2 * lane;
#pragma unroll
                    for (int q = 0; q < Q; q++) {
                        int2 v = make_int2(-1, -1);
                        if (q < nq) v = *reinterpret_cast<const int2 *>(idl + q * 64);
                        id[0][q][0] = v.x;
                        id[0][q][1] = v.y;
#pragma unroll
                        for (int i = 0; i < 2; i++)  // exception rows (id < 0) are computed as full rows and not stored
                            mk[0][q][i] = id[0][q][i] >= 0 ? s_masks[id[0][q][i]] : kFullBox;
                        zl[0][q] = mk[0][q][0] == (kFullBox & ~kLBits);
                        zr[0][q] = mk[0][q][1] == (kFullBox & ~kRBits);
                        other = other || !(mk[0][q][0] == kFullBox || zl[0][q]) || !(mk[0][q][1] == kFullBox || zr[0][q]);
                        anyl = anyl || zl[0][q];
                        anyr = anyr || zr[0][q];
                    }
                    double acc[1][Q][2];
                    const unsigned vote = __ballot_sync(0xffffffffu, other) ? 4u
                                          : ((__ballot_sync(0xffffffffu, anyl) ? 1u : 0u) | (__ballot_sync(0xffffffffu, anyr) ? 2u : 0u));
                    if (vote == 0) box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, false, false>(w, k, mk, zl, zr, vc, vo, acc);
                    else if (vote == 1) box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, true, false>(w, k, mk, zl, zr, vc, vo, acc);
                    else if (vote == 2) box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, false, true>(w, k, mk, zl, zr, vc, vo, acc);
                    else {
                        box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 1, false, false>(w, k, mk, zl, zr, vc, vo, acc);
#pragma unroll
                        for (int q = 0; q < Q; q++)
#pragma unroll
                            for (int i = 0; i < 2; i++)  // patterns outside the box: List 1 per lane
                                if (mk[0][q][i] == kGenericMask)
                                    acc[0][q][i] = pattern_row(p, p.disp, p.ends, p.table, id[0][q][i],
                                                               xi_c + (int64_t)(pw + q) * sz64 + (int64_t)j * sy64 + 2 * lane + i);
                    }
#pragma unroll
                    for (int q = 0; q < Q; q++) {
                        double *dst = yw + (q * sz + j * sy);
                        if (id[0][q][0] >= 0 && id[0][q][1] >= 0)
                            *reinterpret_cast<double2 *>(dst) = make_double2(acc[0][q][0], acc[0][q][1]);
                        else {
                            if (id[0][q][0] >= 0) dst[0] = acc[0][q][0];
                            if (id[0][q][1] >= 0) dst[1] = acc[0][q][1];
                        }
                    }
                }
            }
        }
    }
    cp_async_wait<0>();
}

// -----------------------------------------------------------------------------
// Sliding-window kernel, wide tile ("box6"): NX adjacent columns (4 or 8) and Q planes
// per thread, one line per step.  With NX = 8 a warp spans 256 columns: the per-step
// setup is amortised over 8 rows per thread, only 2 of the NX/2+2 loads per (line,
// plane) are halo loads, and the x-boundary rows are always the first / last column
// of a thread, so ONE chain variant serves every warp: the nine dx=-1 operands of the
// first column and the nine dx=+1 operands of the last column are selected per lane
// (zeroed when that row's mask lacks exactly those entries).  Any other partial mask
// in the step takes the fully masked chain.  NX*Q independent chains per thread.
// -----------------------------------------------------------------------------
template <int NX, int Q, bool OFF_NEG1, int CENTER_POS, bool MASKED>
__device__ __forceinline__ void box6_chain(const double (&w)[3][Q + 2][NX + 2], int kb, const uint32_t (&mk)[Q][NX],
                                           const bool (&zl)[Q], const bool (&zr)[Q], double vc, double vo,
                                           double (&acc)[Q][NX]) {
    double hl[Q][3][3], hr[Q][3][3];
    if (!MASKED) {
#pragma unroll
        for (int q = 0; q < Q; q++)
#pragma unroll
            for (int dz = 0; dz < 3; dz++)
#pragma unroll
                for (int dy = 0; dy < 3; dy++) {
                    const int s = (kb + dy + 2) % 3;
                    hl[q][dz][dy] = zl[q] ? 0.0 : w[s][q + dz][0];
                    hr[q][dz][dy] = zr[q] ? 0.0 : w[s][q + dz][NX + 1];
                }
    }
#pragma unroll
    for (int q = 0; q < Q; q++)
#pragma unroll
        for (int i = 0; i < NX; i++) acc[q][i] = 0.0;
    auto centre = [&]() {
#pragma unroll
        for (int q = 0; q < Q; q++)
#pragma unroll
            for (int i = 0; i < NX; i++) {
                const double pr = __dmul_rn(vc, w[kb % 3][q + 1][i + 1]);
                acc[q][i] = __dadd_rn(acc[q][i], (MASKED && !(mk[q][i] >> 13 & 1u)) ? 0.0 : pr);
            }
    };
    if (CENTER_POS == 0) centre();
#pragma unroll
    for (int t = 0; t < 27; t++) {
        if (t == 13 && CENTER_POS != 2) continue;
        const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
#pragma unroll
        for (int q = 0; q < Q; q++)
#pragma unroll
            for (int i = 0; i < NX; i++) {
                double e = w[(kb + dy + 2) % 3][q + dz][i + dx];
                if (!MASKED && i + dx == 0) e = hl[q][dz][dy];
                if (!MASKED && i + dx == NX + 1) e = hr[q][dz][dy];
                if (OFF_NEG1) {
                    if (MASKED) e = (mk[q][i] >> t & 1u) ? e : 0.0;
                    acc[q][i] = __dsub_rn(acc[q][i], e);
                } else {
                    double pr = __dmul_rn(vo, e);
                    if (MASKED) pr = (mk[q][i] >> t & 1u) ? pr : 0.0;
                    acc[q][i] = __dadd_rn(acc[q][i], pr);
                }
            }
    }
    if (CENTER_POS == 1) centre();
}

struct Box6Smem {
    uint32_t cls0, cls1, clsm, masks;  // 32-bit shared addresses (tables indexed by id + 1)
};

template <int NX, int Q, bool OFF_NEG1, int CENTER_POS>
__device__ __forceinline__ void box6_march(const PatternArgs &p, const Box6Smem sm, const double *__restrict__ xw,
                                           const int32_t *__restrict__ idw, double *__restrict__ yw, int64_t xi_w, int lane,
                                           int nb, bool lane_ok, int nq) {
    constexpr int P = Q + 2, WX = NX + 2;
    const int sy = p.sy;
    const int sz = sy * p.plane_lines;
    const int lo = lane * NX;
    double w[3][P][WX];
    auto load_line = [&](int slot, int line_off) {
#pragma unroll
        for (int pz = 0; pz < P; pz++) {
            const double *pl = xw + (lo + (pz - 1) * sz + line_off);
            w[slot][pz][0] = __ldg(pl - 1);
#pragma unroll
            for (int h = 0; h < NX / 2; h++) {
                const double2 v = __ldg(reinterpret_cast<const double2 *>(pl) + h);
                w[slot][pz][1 + 2 * h] = v.x;
                w[slot][pz][2 + 2 * h] = v.y;
            }
            w[slot][pz][NX + 1] = __ldg(pl + NX);
        }
    };
    bool vq[Q];
#pragma unroll
    for (int q = 0; q < Q; q++) vq[q] = lane_ok && q < nq;
    auto load_ids = [&](int q, bool line_ok, int line_off, int (&out)[NX]) {
#pragma unroll
        for (int i = 0; i < NX; i++) out[i] = -1;  // rows outside the tile: computed, never stored
        if (vq[q] && line_ok) {
            const int4 *ptr = reinterpret_cast<const int4 *>(idw + (lo + q * sz + line_off));
#pragma unroll
            for (int h = 0; h < NX / 4; h++) {
                const int4 v = ld_stream(ptr + h);
                out[4 * h] = v.x; out[4 * h + 1] = v.y; out[4 * h + 2] = v.z; out[4 * h + 3] = v.w;
            }
        }
    };
    load_line(2, -sy);
    load_line(0, 0);
    int idn[Q][NX];
#pragma unroll
    for (int q = 0; q < Q; q++) load_ids(q, 0 < nb, 0, idn[q]);
    const int pf = p.prefetch * sy;
    const double vc = p.v_center, vo = p.v_off;
#pragma unroll 1
    for (int j0 = 0; j0 < nb; j0 += 3) {
#pragma unroll
        for (int kb = 0; kb < 3; kb++) {
            const int j = j0 + kb;
            if (j < nb) {
                load_line((kb + 1) % 3, sy);
                int id[Q][NX];
                uint32_t other = 0;
                bool zl[Q], zr[Q];
#pragma unroll
                for (int q = 0; q < Q; q++) {
#pragma unroll
                    for (int i = 0; i < NX; i++) id[q][i] = idn[q][i];
                    load_ids(q, j + 1 < nb, sy, idn[q]);
                    const uint32_t c0 = lds_u32(sm.cls0 + 4 + 4 * id[q][0]);
                    const uint32_t c1 = lds_u32(sm.cls1 + 4 + 4 * id[q][NX - 1]);
                    zl[q] = c0 & 1u;
                    zr[q] = c1 & 2u;
                    other |= c0 | c1;
#pragma unroll
                    for (int i = 1; i < NX - 1; i++) other |= lds_u32(sm.clsm + 4 + 4 * id[q][i]);
                }
                if (pf > 0 && (lane & 1) == 0) {  // lines `prefetch` steps ahead, HBM -> L2 (one request per 128 bytes)
#pragma unroll
                    for (int q = 0; q < Q; q++) {
                        prefetch_l2(xw + (lo + q * sz + pf));
                        if ((lane & 3) == 0) prefetch_l2(idw + (lo + q * sz + pf));
                    }
                }
                double acc[Q][NX];
                uint32_t mk[Q][NX];
                if (!__any_sync(0xffffffffu, (other & 4u) != 0)) {
                    box6_chain<NX, Q, OFF_NEG1, CENTER_POS, false>(w, kb, mk, zl, zr, vc, vo, acc);
                } else {
#pragma unroll
                    for (int q = 0; q < Q; q++)
#pragma unroll
                        for (int i = 0; i < NX; i++) mk[q][i] = lds_u32(sm.masks + 4 + 4 * id[q][i]);
                    box6_chain<NX, Q, OFF_NEG1, CENTER_POS, true>(w, kb, mk, zl, zr, vc, vo, acc);
#pragma unroll
                    for (int q = 0; q < Q; q++)
#pragma unroll
                        for (int i = 0; i < NX; i++)  // patterns outside the box: List 1 per lane
                            if (mk[q][i] == kGenericMask)
                                acc[q][i] = pattern_row_cold(p, id[q][i], xi_w + lo + q * (int64_t)sz + i);
                }
#pragma unroll
                for (int q = 0; q < Q; q++) {
                    double *dst = yw + (lo + q * sz);
                    int all = id[q][0];
#pragma unroll
                    for (int i = 1; i < NX; i++) all |= id[q][i];
                    if (all >= 0) {
#pragma unroll
                        for (int h = 0; h < NX / 2; h++)
                            reinterpret_cast<double2 *>(dst)[h] = make_double2(acc[q][2 * h], acc[q][2 * h + 1]);
                    } else {
#pragma unroll
                        for (int i = 0; i < NX; i++)
                            if (id[q][i] >= 0) dst[i] = acc[q][i];
                    }
                }
                xw += sy;
                idw += sy;
                yw += sy;
                xi_w += sy;
            }
        }
    }
}

template <int NX, int R, int WC, int Q, int MINB, bool OFF_NEG1, int CENTER_POS>
__global__ void __launch_bounds__(WC * 32, MINB) spmv_pattern_box6_kernel(PatternArgs p, int n_planes) {
    constexpr int CW = 32 * NX;  // columns per warp
    __shared__ uint32_t s_cls0[kDictSmemPat + 1], s_cls1[kDictSmemPat + 1], s_clsm[kDictSmemPat + 1], s_masks1[kDictSmemPat + 1];
    for (int i = threadIdx.x; i <= p.n_patterns; i += WC * 32) {
        const uint32_t m = i == 0 ? kFullBox : p.masks[i - 1];
        s_masks1[i] = m;
        s_cls0[i] = m == kFullBox ? 0u : (m == (kFullBox & ~kLBits) ? 1u : 4u);
        s_cls1[i] = m == kFullBox ? 0u : (m == (kFullBox & ~kRBits) ? 2u : 4u);
        s_clsm[i] = m == kFullBox ? 0u : 4u;
    }
    __syncthreads();
    Box6Smem sm;
    sm.cls0 = (uint32_t)__cvta_generic_to_shared(s_cls0);
    sm.cls1 = (uint32_t)__cvta_generic_to_shared(s_cls1);
    sm.clsm = (uint32_t)__cvta_generic_to_shared(s_clsm);
    sm.masks = (uint32_t)__cvta_generic_to_shared(s_masks1);
    const uint32_t *s_masks = s_masks1 + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int a_w = blockIdx.x * CW;
    const int c0 = (blockIdx.z * WC + warp) * Q;
    const int b0 = blockIdx.y * R;
    if (c0 >= n_planes) return;
    const int nb = min(R, p.plane_lines - b0);
    const int nq = min(Q, n_planes - c0);
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sy = p.sy, sz = sy * p.plane_lines;
    const int64_t r_w = a_w + sy * (b0 + (int64_t)p.plane_lines * c0);
    if (r_w >= n_rows) return;
    const int cols_ok = min(CW, p.sy - a_w);  // a multiple of NX (launcher guarantees sy % NX == 0)
    const int64_t xi_w = p.g0 + p.row_begin + r_w;
    const int pf = p.prefetch > 0 ? p.prefetch : 0;
    const int64_t last_row = r_w + (cols_ok - 1) + (int64_t)(nb - 1) * sy + (int64_t)(nq - 1) * sz;
    const int64_t x_lo = xi_w - sy - sz - 1;
    const int64_t x_hi = xi_w + CW + (int64_t)(nb + 1 + pf) * sy + (int64_t)Q * sz + 1;
    const int64_t id_hi = r_w + CW + (int64_t)(nb + 1 + pf) * sy + (int64_t)(nq - 1) * sz;
    const bool interior = last_row < n_rows && x_lo >= 0 && x_hi < p.x_len && id_hi <= n_rows + 1024;
    if (interior) {
        box6_march<NX, Q, OFF_NEG1, CENTER_POS>(p, sm, p.x + xi_w, p.ids + p.row_begin + r_w, p.y + p.row_begin + r_w, xi_w, lane,
                                                nb, lane * NX + NX - 1 < cols_ok, nq);
    } else {
#pragma unroll 1
        for (int part = 0; part < NX; part++)  // guarded one-column march of the v2 kernel, 32 columns at a time
            box_march<Q, 0, OFF_NEG1, CENTER_POS, true>(p, s_masks, r_w + part * 32 + lane, nb, n_rows, nq,
                                                        part * 32 + lane < cols_ok, false, false);
    }
}

// -----------------------------------------------------------------------------
// Sliding-window kernel, software-pipelined ring ("box7").
// Measured regime of box3/box5 (profiles/): each warp spends ~90% of a step outside its
// FP64 chain, on a serial setup (window loads -> ids -> class lookup -> vote -> branch)
// whose latencies are exposed because only ~10 warps fit per SM (96-register window).
// Here the setup of step j+1 is issued in the SAME basic block as the DADD chain of
// step j -- the chain occupies every other issue slot (DADD issues once per 2 cycles),
// the setup's shared-memory loads, class lookups, halo selects and the vote fill the
// rest -- and everything the setup reads comes from a cp.async shared-memory ring
// filled DEPTH lines ahead (box5), so no global latency is on the path at all.
//   * window: 4 slots (lines j-1, j, j+1 in use, j+2 arriving) x (Q+2) planes x 4 cols
//   * one chain variant for every warp: the nine dx=-1 operands of the left column and
//     the nine dx=+1 operands of the right column are selected per lane (zeroed for rows
//     whose mask lacks exactly those entries); a step with any other partial mask runs
//     the fully masked chain (same basic-block structure, rare).
// -----------------------------------------------------------------------------
template <int R, int WC, int Q, int DEPTH, int MINB, bool OFF_NEG1, int CENTER_POS>
__global__ void __launch_bounds__(WC * 32, MINB) spmv_pattern_box7_kernel(PatternArgs p, int n_planes) {
    constexpr int T = WC * 32;
    constexpr int NP = WC * Q;
    constexpr int XP = NP + 2;
    constexpr int XW = 68;
    constexpr int XCH = XP * (XW / 2);
    constexpr int ICH = NP * 16;
    constexpr int NCH = XCH + ICH;
    constexpr int PER = (NCH + T - 1) / T;
    constexpr int S = 4, P = Q + 2;
    static_assert(DEPTH >= 4, "ring depth");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *xs = reinterpret_cast<double *>(smem_raw);                                   // [DEPTH][XP][XW]
    int32_t *is = reinterpret_cast<int32_t *>(smem_raw + (size_t)DEPTH * XP * XW * 8);   // [DEPTH][NP][64]
    __shared__ uint32_t s_cls0[kDictSmemPat + 1], s_cls1[kDictSmemPat + 1], s_masks1[kDictSmemPat + 1];
    box3_fill_tables(p, s_cls0, s_cls1, s_masks1, threadIdx.x, T);
    const uint32_t cls0_a = (uint32_t)__cvta_generic_to_shared(s_cls0);
    const uint32_t cls1_a = (uint32_t)__cvta_generic_to_shared(s_cls1);
    const uint32_t mask_a = (uint32_t)__cvta_generic_to_shared(s_masks1);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int a_w = blockIdx.x * 64;
    const int c0 = blockIdx.z * NP;
    const int b0 = blockIdx.y * R;
    const int nb = min(R, p.plane_lines - b0);
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sy64 = p.sy, sz64 = sy64 * p.plane_lines;
    const int64_t r_c = a_w + sy64 * (b0 + (int64_t)p.plane_lines * c0);
    const int cols_ok = min(64, p.sy - a_w);
    const int nq_cta = min(NP, n_planes - c0);
    const int64_t xi_c = p.g0 + p.row_begin + r_c;
    const int64_t x_lo = xi_c - sy64 - sz64 - 2;
    const int64_t x_hi = xi_c + 66 + (int64_t)nb * sy64 + (int64_t)NP * sz64;
    const int64_t last_row = r_c + (cols_ok - 1) + (int64_t)(nb - 1) * sy64 + (int64_t)(nq_cta - 1) * sz64;
    const bool interior = x_lo >= 0 && x_hi < p.x_len && last_row < n_rows && cols_ok == 64;
    __syncthreads();
    if (!interior) {  // CTA-uniform: grid edges, slab ends, ragged ranges -> guarded v2 march
        const int cw = c0 + warp * Q;
        if (cw < n_planes && r_c + (int64_t)warp * Q * sz64 < n_rows)
            box3_edge_tile<Q, OFF_NEG1, CENTER_POS>(p, s_masks1 + 1, r_c + (int64_t)warp * Q * sz64, lane, nb, n_rows,
                                                    min(Q, n_planes - cw), cols_ok);
        return;
    }
    const int sy = p.sy, sz = sy * p.plane_lines;
    const double *xg = p.x + xi_c;
    const int32_t *ig = p.ids + p.row_begin + r_c;
    int src_off[PER];
    uint32_t dst_off[PER];
    int kind[PER];
    const uint32_t xs_base = (uint32_t)__cvta_generic_to_shared(xs);
    const uint32_t is_base = (uint32_t)__cvta_generic_to_shared(is);
#pragma unroll
    for (int k = 0; k < PER; k++) {
        const int c = threadIdx.x + k * T;
        if (c < XCH) {
            const int pz = c / (XW / 2), j = c % (XW / 2);
            kind[k] = 0;
            src_off[k] = (pz - 1) * sz - 2 + 2 * j;
            dst_off[k] = (uint32_t)((pz * XW + 2 * j) * 8);
        } else if (c < NCH) {
            const int q = (c - XCH) / 16, j = (c - XCH) % 16;
            kind[k] = q < nq_cta ? 1 : 2;
            src_off[k] = q * sz + 4 * j;
            dst_off[k] = (uint32_t)((q * 64 + 4 * j) * 4);
        } else {
            kind[k] = 2; src_off[k] = 0; dst_off[k] = 0;
        }
    }
    auto fetch = [&](int line) {  // stage line `line` (-1 .. nb) into ring slot (line+1) % DEPTH; always one group
        if (line <= nb) {
            const int slot = (line + 1) % DEPTH;
#pragma unroll
            for (int k = 0; k < PER; k++) {
                if (kind[k] == 0)
                    cp_async16(xs_base + (uint32_t)(slot * XP * XW * 8) + dst_off[k], xg + (src_off[k] + line * sy));
                else if (kind[k] == 1 && line >= 0 && line < nb)
                    cp_async16(is_base + (uint32_t)(slot * NP * 64 * 4) + dst_off[k], ig + (src_off[k] + line * sy));
            }
        }
        cp_async_commit();
    };
    const int pw = warp * Q;
    const int nq = min(Q, n_planes - (c0 + pw));  // <= 0: this warp only helps with the copies
    double w[S][P][4];
    auto load_line = [&](int wslot, int line) {
        const double *base = xs + ((line + 1) % DEPTH) * (XP * XW) + pw * XW + 2 * lane;
#pragma unroll
        for (int pz = 0; pz < P; pz++) {
            const double *pl = base + pz * XW;
            const double2 v = *reinterpret_cast<const double2 *>(pl + 2);
            w[wslot][pz][0] = pl[1];
            w[wslot][pz][1] = v.x;
            w[wslot][pz][2] = v.y;
            w[wslot][pz][3] = pl[4];
        }
    };
    // ids of line `line` -> per-row ids, halo-select flags and the "other mask" flag of that line
    auto classify = [&](int line, int (&id)[Q][2], bool (&zl)[Q], bool (&zr)[Q]) -> uint32_t {
        uint32_t other = 0;
        const int32_t *idl = is + ((line + 1) % DEPTH) * (NP * 64) + pw * 64 + 2 * lane;
#pragma unroll
        for (int q = 0; q < Q; q++) {
            int2 v = make_int2(-1, -1);
            if (q < nq && line < nb) v = *reinterpret_cast<const int2 *>(idl + q * 64);
            id[q][0] = v.x;
            id[q][1] = v.y;
            const uint32_t c0v = lds_u32(cls0_a + 4 + 4 * v.x), c1v = lds_u32(cls1_a + 4 + 4 * v.y);
            zl[q] = c0v & 1u;
            zr[q] = c1v & 2u;
            other |= (c0v | c1v) & 4u;
        }
        return other;
    };
#pragma unroll
    for (int l = -1; l < DEPTH - 1; l++) fetch(l);  // lines -1 .. DEPTH-2 in flight
    cp_async_wait<DEPTH - 3>();                     // lines -1, 0, 1 have landed
    __syncthreads();
    load_line(S - 1, -1);
    load_line(0, 0);
    load_line(1, 1);
    int id[Q][2];
    bool zl[Q], zr[Q];
    bool slow = __any_sync(0xffffffffu, classify(0, id, zl, zr) != 0);
    double *yw = p.y + p.row_begin + r_c + (int64_t)pw * sz64 + 2 * lane;
    const double vc = p.v_center, vo = p.v_off;
    const int pf = (x_hi + (int64_t)(DEPTH + p.prefetch) * sy64 < p.x_len &&
                    last_row + (int64_t)(DEPTH + p.prefetch) * sy64 < n_rows) ? p.prefetch : 0;
#pragma unroll 1
    for (int j0 = 0; j0 < nb; j0 += S) {
#pragma unroll
        for (int k = 0; k < S; k++) {
            const int j = j0 + k;
            if (j < nb) {  // CTA-uniform
                cp_async_wait<DEPTH - 4>();  // line j+2 has landed (groups up to line j+DEPTH-2 are committed)
                __syncthreads();
                fetch(j + DEPTH - 1);
                if (pf > 0 && lane < 8) {  // further ahead: HBM -> L2, one request per 128-byte line
                    const int line = j + DEPTH - 1 + pf;
#pragma unroll
                    for (int q = 0; q < Q; q++) {
                        prefetch_l2(xg + ((pw + q) * sz + line * sy + 16 * lane));
                        if (lane < 2) prefetch_l2(ig + ((pw + q) * sz + line * sy + 32 * lane));
                    }
                    if (warp == 0) prefetch_l2(xg + (-sz + line * sy + 16 * lane));
                    if (warp == WC - 1) prefetch_l2(xg + (NP * sz + line * sy + 16 * lane));
                }
                int idn[Q][2];
                bool zln[Q], zrn[Q];
                uint32_t other_n;
                double acc[1][Q][2];
                uint32_t mk[1][Q][2];
                bool zl1[1][Q], zr1[1][Q];
#pragma unroll
                for (int q = 0; q < Q; q++) { zl1[0][q] = zl[q]; zr1[0][q] = zr[q]; }
                // Slot of line l is (l mod 4) with line -1 in slot 3: chain(j) reads slots k-1, k, k+1; line j+2 -> slot k+2.
                if (false) {  // ablation: no chain (profiles/r01_ablation_nochain.log)
                    load_line((k + 2) % S, j + 2);
                    other_n = classify(j + 1, idn, zln, zrn);
#pragma unroll
                    for (int q = 0; q < Q; q++)
#pragma unroll
                        for (int i = 0; i < 2; i++) acc[0][q][i] = w[k][q + 1][i + 1] + w[(k + 1) % S][q + 2][i + 2];
                } else if (!slow) {
                    load_line((k + 2) % S, j + 2);             // setup of step j+1 ...
                    other_n = classify(j + 1, idn, zln, zrn);
                    box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, true, true>(w, k, mk, zl1, zr1, vc, vo, acc);  // ... under chain j
                } else {
                    load_line((k + 2) % S, j + 2);
                    other_n = classify(j + 1, idn, zln, zrn);
#pragma unroll
                    for (int q = 0; q < Q; q++)
#pragma unroll
                        for (int i = 0; i < 2; i++) mk[0][q][i] = lds_u32(mask_a + 4 + 4 * id[q][i]);
                    box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 1, false, false>(w, k, mk, zl1, zr1, vc, vo, acc);
#pragma unroll
                    for (int q = 0; q < Q; q++)
#pragma unroll
                        for (int i = 0; i < 2; i++)  // patterns outside the box: List 1 per lane
                            if (mk[0][q][i] == kGenericMask)
                                acc[0][q][i] = pattern_row_cold(p, id[q][i], xi_c + (int64_t)(pw + q) * sz64 + (int64_t)j * sy64 + 2 * lane + i);
                }
#pragma unroll
                for (int q = 0; q < Q; q++) {
                    double *dst = yw + (q * sz + j * sy);
                    if ((id[q][0] | id[q][1]) >= 0) *reinterpret_cast<double2 *>(dst) = make_double2(acc[0][q][0], acc[0][q][1]);
                    else {
                        if (id[q][0] >= 0) dst[0] = acc[0][q][0];
                        if (id[q][1] >= 0) dst[1] = acc[0][q][1];
                    }
                }
#pragma unroll
                for (int q = 0; q < Q; q++) {
                    id[q][0] = idn[q][0]; id[q][1] = idn[q][1];
                    zl[q] = zln[q]; zr[q] = zrn[q];
                }
                slow = __any_sync(0xffffffffu, other_n != 0);
            }
        }
    }
    cp_async_wait<0>();
}

// -----------------------------------------------------------------------------
// Sliding-window kernel, warp-specialised TMA ring ("box8").
// What the measurements of box3 / box5 / box7 say: the direct-load
// march is bound by memory-level parallelism (about 16 KB in flight per SM, every
// memory unit below 35% busy), and the cp.async rings fix that but load every thread
// with copy bookkeeping and a CTA barrier per line, so they become instruction bound.
// Here the roles are split:
//   * producer: lane 0 of warp 0 walks the CTA's tiles and, per grid line, issues one
//     TMA bulk copy (cp.async.bulk, SASS UBLKCP) per staged x plane (2080 contiguous
//     bytes: 256 columns + halo) and per id plane (1024 bytes) into a DEPTH-deep
//     shared-memory ring; completion is counted on an mbarrier per stage (complete_tx).
//   * consumers: 12 warps = 4 across x (64 columns each) x 3 across z (Q = 2 planes
//     each).  Per line: wait on the stage's "full" mbarrier, refill the register window
//     from shared memory, classify the rows from their pattern ids, run box3's chains
//     in the dictionary's order, store y, release the stage on its "empty" mbarrier.
//     No global loads, no copy instructions, no CTA-wide barrier on that path.
// Persistent grid (one CTA per SM, tiles round-robin).  Tiles that are not interior
// (staged range leaves x, partial width, ragged rows) are served by the guarded v2
// march on the consumer warps.  Needs sy % 256 == 0-style alignment (checked by the
// launcher); everything else falls back to box3.
// -----------------------------------------------------------------------------
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

template <int R, int DEPTH, int WZ, bool OFF_NEG1, int CENTER_POS>
__global__ void __maxnreg__(WZ == 3 ? 128 : 168) spmv_pattern_box8_kernel(PatternArgs p, int n_planes, int n_tiles_y,
                                                                      int n_tiles_z, int n_tiles_x) {
    constexpr int Q = 2, WA = 4, NCW = WA * WZ, NT = (1 + NCW) * 32;
    constexpr int NP = WZ * Q;        // planes computed per tile
    constexpr int XP = NP + 2;        // x planes staged
    constexpr int XW = 256 + 4;       // staged doubles per x line: columns a_c-2 .. a_c+257
    constexpr int XSTAGE = XP * XW;   // doubles
    constexpr int ISTAGE = NP * 256;  // ints
    constexpr uint32_t STAGE_BYTES = XSTAGE * 8 + ISTAGE * 4;
    constexpr int S = 3, P = Q + 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[DEPTH], empty_bar[DEPTH];
    __shared__ uint32_t s_cls0[kDictSmemPat + 1], s_cls1[kDictSmemPat + 1], s_masks1[kDictSmemPat + 1];
    box3_fill_tables(p, s_cls0, s_cls1, s_masks1, threadIdx.x, NT);
    if (threadIdx.x == 0) {
        for (int s = 0; s < DEPTH; s++) {
            mbar_init(smem_u32(&full_bar[s]), 1);
            mbar_init(smem_u32(&empty_bar[s]), NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sy64 = p.sy, sz64 = sy64 * p.plane_lines;
    const int sy = p.sy, sz = sy * p.plane_lines;
    const int n_tiles = n_tiles_x * n_tiles_y * n_tiles_z;

    // Tile geometry, identical for producer and consumers.
    struct Tile {
        int a_c, b0, c0, nb, nq;
        int64_t r_c, xi_c;
        bool interior;
    };
    auto tile_of = [&](int t) {
        Tile T;
        const int tx = t % n_tiles_x, ty = (t / n_tiles_x) % n_tiles_y, tz = t / (n_tiles_x * n_tiles_y);
        T.a_c = tx * 256;
        T.b0 = ty * R;
        T.c0 = tz * NP;
        T.nb = min(R, p.plane_lines - T.b0);
        T.nq = min(NP, n_planes - T.c0);
        T.r_c = T.a_c + sy64 * (T.b0 + (int64_t)p.plane_lines * T.c0);
        T.xi_c = p.g0 + p.row_begin + T.r_c;
        const int cols_ok = min(256, p.sy - T.a_c);
        const int64_t x_lo = T.xi_c - sy64 - sz64 - 2;
        const int64_t x_hi = T.xi_c + 258 + (int64_t)T.nb * sy64 + (int64_t)T.nq * sz64;
        const int64_t last_row = T.r_c + (cols_ok - 1) + (int64_t)(T.nb - 1) * sy64 + (int64_t)(T.nq - 1) * sz64;
        T.interior = cols_ok == 256 && x_lo >= 0 && x_hi < p.x_len && last_row < n_rows;
        return T;
    };

    if (warp == 0) {
        // ------------------------------------------------------------------ producer
        if (lane != 0) return;
        int it = 0;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
            const Tile T = tile_of(t);
            if (!T.interior) continue;
            const double *xg = p.x + T.xi_c;
            const int32_t *ig = p.ids + p.row_begin + T.r_c;
            for (int line = -1; line <= T.nb; line++, it++) {
                const int s = it % DEPTH, n = it / DEPTH;
                if (n > 0) mbar_wait(smem_u32(&empty_bar[s]), (n - 1) & 1);  // consumers released the previous use
                const bool with_ids = line >= 0 && line < T.nb;
                const uint32_t bar = smem_u32(&full_bar[s]);
                const uint32_t dst = smem_u32(smem_raw + (size_t)s * STAGE_BYTES);
                mbar_expect_tx(bar, (uint32_t)(T.nq + 2) * XW * 8 + (with_ids ? (uint32_t)T.nq * 1024 : 0u));
                for (int pz = 0; pz < T.nq + 2; pz++)
                    bulk_g2s(dst + pz * XW * 8, xg + ((int64_t)(pz - 1) * sz + (int64_t)line * sy - 2), XW * 8, bar);
                if (with_ids)
                    for (int q = 0; q < T.nq; q++)
                        bulk_g2s(dst + XSTAGE * 8 + q * 1024, ig + ((int64_t)q * sz + (int64_t)line * sy), 1024, bar);
            }
        }
        return;
    }
    // ---------------------------------------------------------------------- consumers
    const int cw = warp - 1;
    const int xw_i = cw % WA, zw = cw / WA;
    const int pw = zw * Q;  // first plane (within the tile) of this warp
    Box3Smem sm;
    sm.cls0 = smem_u32(s_cls0);
    sm.cls1 = smem_u32(s_cls1);
    sm.masks = smem_u32(s_masks1);
    const double vc = p.v_center, vo = p.v_off;
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const Tile T = tile_of(t);
        if (!T.interior) {  // grid edges, slab ends, ragged ranges: guarded v2 march, 64 columns per warp
            const int cwz = T.c0 + pw;
            const int cols_ok = min(64, p.sy - (T.a_c + 64 * xw_i));
            if (cwz < n_planes && cols_ok > 0 && T.r_c + 64 * xw_i + (int64_t)pw * sz64 < n_rows)
                box3_edge_tile<Q, OFF_NEG1, CENTER_POS>(p, s_masks1 + 1, T.r_c + 64 * xw_i + (int64_t)pw * sz64, lane, T.nb, n_rows,
                                                        min(Q, n_planes - cwz), cols_ok);
            continue;
        }
        const int nq = min(Q, T.nq - pw);  // <= 0: this warp only keeps the ring protocol going
        double w[S][P][4];
        auto wait_full = [&](int i) { mbar_wait(smem_u32(&full_bar[i % DEPTH]), (i / DEPTH) & 1); };
        auto release = [&](int i) {
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&empty_bar[i % DEPTH]));
        };
        auto load_line = [&](int wslot, int i) {  // window slot <- x line held by ring entry i
            const double *base = reinterpret_cast<const double *>(smem_raw + (size_t)(i % DEPTH) * STAGE_BYTES) + pw * XW + 64 * xw_i + 2 * lane;
#pragma unroll
            for (int pz = 0; pz < P; pz++) {
                const double *pl = base + pz * XW;
                const double2 v = *reinterpret_cast<const double2 *>(pl + 2);
                w[wslot][pz][0] = pl[1];
                w[wslot][pz][1] = v.x;
                w[wslot][pz][2] = v.y;
                w[wslot][pz][3] = pl[4];
            }
        };
        // lines -1 and 0
        wait_full(it);
        if (nq > 0) load_line(S - 1, it);
        release(it);
        wait_full(it + 1);
        if (nq > 0) load_line(0, it + 1);
        double *yw = p.y + p.row_begin + T.r_c + (int64_t)pw * sz64 + 64 * xw_i + 2 * lane;
        const int64_t xi_w = T.xi_c + (int64_t)pw * sz64 + 64 * xw_i;
#pragma unroll 1
        for (int j0 = 0; j0 < T.nb; j0 += S) {
#pragma unroll
            for (int k = 0; k < S; k++) {
                const int j = j0 + k;
                if (j < T.nb) {
                    const int ej = it + 1 + j;  // ring entry of line j; line j+1 is entry ej + 1
                    wait_full(ej + 1);
                    if (nq > 0) {
                        load_line((k + 1) % S, ej + 1);
                        const int32_t *idl = reinterpret_cast<const int32_t *>(smem_raw + (size_t)(ej % DEPTH) * STAGE_BYTES + XSTAGE * 8) +
                                             pw * 256 + 64 * xw_i + 2 * lane;
                        int id[1][Q][2];
                        uint32_t c0v[Q], c1v[Q], wv = 0;
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            int2 v = make_int2(-1, -1);
                            if (q < nq) v = *reinterpret_cast<const int2 *>(idl + q * 256);
                            id[0][q][0] = v.x;
                            id[0][q][1] = v.y;
                            c0v[q] = lds_u32(sm.cls0 + 4 + 4 * v.x);
                            c1v[q] = lds_u32(sm.cls1 + 4 + 4 * v.y);
                            wv |= c0v[q] | c1v[q];
                        }
                        release(ej);  // x of line j was consumed one step ago, its ids just now
                        double acc[1][Q][2];
                        uint32_t mk[1][Q][2];
                        bool zl[1][Q], zr[1][Q];
                        const unsigned vote = __reduce_or_sync(0xffffffffu, wv);
                        if (vote == 0) {
                            box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, false, false>(w, k, mk, zl, zr, vc, vo, acc);
                        } else if (vote == 1 || vote == 2) {
#pragma unroll
                            for (int q = 0; q < Q; q++) { zl[0][q] = c0v[q] != 0; zr[0][q] = c1v[q] != 0; }
                            if (vote == 1) box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, true, false>(w, k, mk, zl, zr, vc, vo, acc);
                            else box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, false, true>(w, k, mk, zl, zr, vc, vo, acc);
                        } else {
#pragma unroll
                            for (int q = 0; q < Q; q++)
#pragma unroll
                                for (int i = 0; i < 2; i++) mk[0][q][i] = lds_u32(sm.masks + 4 + 4 * id[0][q][i]);
                            box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 1, false, false>(w, k, mk, zl, zr, vc, vo, acc);
#pragma unroll
                            for (int q = 0; q < Q; q++)
#pragma unroll
                                for (int i = 0; i < 2; i++)  // patterns outside the box: List 1 per lane
                                    if (mk[0][q][i] == kGenericMask)
                                        acc[0][q][i] = pattern_row_cold(p, id[0][q][i], xi_w + q * sz64 + (int64_t)j * sy64 + 2 * lane + i);
                        }
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            double *dst = yw + (q * sz + j * sy);
                            if ((id[0][q][0] | id[0][q][1]) >= 0) *reinterpret_cast<double2 *>(dst) = make_double2(acc[0][q][0], acc[0][q][1]);
                            else {
                                if (id[0][q][0] >= 0) dst[0] = acc[0][q][0];
                                if (id[0][q][1] >= 0) dst[1] = acc[0][q][1];
                            }
                        }
                    } else {
                        release(ej);
                    }
                }
            }
        }
        release(it + 1 + T.nb);  // the last x line (no ids)
        it += T.nb + 2;
    }
}

// ---- host-side launchers -----------------------------------------------------------
static int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SPMVB_ERR_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
    return SPMVB_OK;
}

static int launch_ell(const double *values, const int32_t *columns, int width, const double *x, int64_t x_col0,
                      double *y, int row_begin, int row_end, const int32_t *row_map, cudaStream_t st) {
    if (row_end <= row_begin || width == 0) {
        if (width == 0 && row_end > row_begin && !row_map)
            SPMVB_CUDA(cudaMemsetAsync(y + row_begin, 0, (size_t)(row_end - row_begin) * 8, st));
        return SPMVB_OK;
    }
    if (options().ell_kernel == 1 && !row_map) {
        const int threads = 128;
        spmv_ell_naive_kernel<<<(row_end - row_begin + threads - 1) / threads, threads, 0, st>>>(
            values, columns, width, x, x_col0, y, row_begin, row_end);
        return check_launch("spmv_ell_naive");
    }
    const int tile0 = row_begin / kTileRows;
    const int tiles = (row_end + kTileRows - 1) / kTileRows - tile0;
    const size_t smem = (size_t)kTileRows * width * 12;
    if (smem > 200 * 1024) return fail(SPMVB_ERR_INVALID_ARGUMENT, "ELL width %d too large for the staged kernel", width);
    if (options().ell_kernel != 2) {
        // TMA bulk pipeline (default): persistent CTAs, NS stages of one tile each
        constexpr int NS = 2;
        const size_t stage = smem;  // multiple of 16 for any width (128 rows)
        const size_t need = stage * NS;
        if (need <= 220 * 1024) {
            static bool tma_attr = false;
            if (!tma_attr) {
                SPMVB_CUDA(cudaFuncSetAttribute(spmv_rows_tma_kernel<kTileRows, NS, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
                tma_attr = true;
            }
            const int per_sm = std::max(1, (int)std::min<size_t>(8, (220 * 1024) / (need + 1024)));
            const int grid = std::min(tiles, 148 * per_sm);
            spmv_rows_tma_kernel<kTileRows, NS, 0><<<grid, kTileRows, need, st>>>(values, columns, nullptr, nullptr, width, 0, x, x_col0, y,
                                                                               row_begin, row_end, tile0, tiles, row_map);
            return check_launch("spmv_ell_tma");
        }
    }
    static bool attr_set = false;
    if (!attr_set) {
        SPMVB_CUDA(cudaFuncSetAttribute(spmv_ell_kernel<kTileRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_set = true;
    }
    spmv_ell_kernel<kTileRows><<<tiles, kTileRows, smem, st>>>(values, columns, width, x, x_col0, y, row_begin,
                                                               row_end, tile0, row_map);
    return check_launch("spmv_ell");
}

static int launch_vt(const spmvb_matrix *a, const double *x, int64_t x_col0, double *y, int row_begin, int row_end,
                     cudaStream_t st) {
    if (row_end <= row_begin) return SPMVB_OK;
    const int tile0 = row_begin / kTileRows;
    const int tiles = (row_end + kTileRows - 1) / kTileRows - tile0;
    const size_t smem = (size_t)kTileRows * (a->width + a->m) * 4 + (size_t)a->m * 8 + 16;
    if (smem > 200 * 1024) return fail(SPMVB_ERR_INVALID_ARGUMENT, "vt width/table too large for the staged kernel");
    if (options().ell_kernel == 3) {  // TMA bulk pipeline: measured slower than the staged kernel for vt (545 vs 470 us)
        constexpr int NS = 2;
        const size_t stage = (size_t)kTileRows * (a->width + a->m) * 4;
        const size_t need = stage * NS;
        if (need <= 200 * 1024) {
            static bool tma_attr = false;
            if (!tma_attr) {
                SPMVB_CUDA(cudaFuncSetAttribute(spmv_rows_tma_kernel<kTileRows, NS, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                tma_attr = true;
            }
            const int per_sm = std::max(1, (int)std::min<size_t>(8, (200 * 1024) / (need + 4096)));
            const int grid = std::min(tiles, 148 * per_sm);
            spmv_rows_tma_kernel<kTileRows, NS, 1><<<grid, kTileRows, need, st>>>(
                nullptr, static_cast<const int32_t *>(a->s[SPMVB_S_SORTED_COLUMNS]), static_cast<const int32_t *>(a->s[SPMVB_S_ENDS]),
                static_cast<const double *>(a->s[SPMVB_S_TABLE]), a->width, a->m, x, x_col0, y, row_begin, row_end, tile0, tiles, nullptr);
            return check_launch("spmv_vt_tma");
        }
    }
    static bool attr_set = false;
    if (!attr_set) {
        SPMVB_CUDA(cudaFuncSetAttribute(spmv_vt_kernel<kTileRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_set = true;
    }
    spmv_vt_kernel<kTileRows><<<tiles, kTileRows, smem, st>>>(
        static_cast<const int32_t *>(a->s[SPMVB_S_SORTED_COLUMNS]), static_cast<const int32_t *>(a->s[SPMVB_S_ENDS]),
        static_cast<const double *>(a->s[SPMVB_S_TABLE]), a->width, a->m, x, x_col0, y, row_begin, row_end, tile0);
    return check_launch("spmv_vt");
}

template <int R, int WC, int Q, int LA>
static int launch_box_rw(const spmvb_matrix *a, PatternArgs &p, cudaStream_t st) {
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    const int n_planes = (int)((n_rows + sz - 1) / sz);
    dim3 grid((p.sy + 31) / 32, (p.plane_lines + R - 1) / R, (n_planes + WC * Q - 1) / (WC * Q));
    dim3 block(WC * 32);
    const bool neg1 = p.v_off == -1.0;
    const int cp = a->box.center_pos;
#define LAUNCH(NEG, CP) spmv_pattern_box_kernel<R, WC, Q, LA, NEG, CP><<<grid, block, 0, st>>>(p, n_planes)
    if (neg1) {
        if (cp == 0) LAUNCH(true, 0); else if (cp == 1) LAUNCH(true, 1); else LAUNCH(true, 2);
    } else {
        if (cp == 0) LAUNCH(false, 0); else if (cp == 1) LAUNCH(false, 1); else LAUNCH(false, 2);
    }
#undef LAUNCH
    return check_launch("spmv_pattern_box");
}

// wide-tile launch: returns 1 when not served
template <int NX, int R, int WC, int Q, int MINB, bool ALLV>
static int launch_box6(const spmvb_matrix *a, PatternArgs &p, cudaStream_t st) {
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    const int n_planes = (int)((n_rows + sz - 1) / sz);
    const bool neg1 = p.v_off == -1.0;
    const int cp = a->box.center_pos;
    if (!ALLV && !(neg1 && cp == 1)) return 1;
    if (p.sy % NX || p.sy % 4 || (p.g0 + p.row_begin) % 4 || p.row_begin % 4 || (uintptr_t)p.ids % 16) return 1;
    dim3 grid((p.sy + 32 * NX - 1) / (32 * NX), (p.plane_lines + R - 1) / R, (n_planes + WC * Q - 1) / (WC * Q));
    dim3 block(WC * 32);
#define LAUNCH6(NEG, CP) spmv_pattern_box6_kernel<NX, R, WC, Q, MINB, NEG, CP><<<grid, block, 0, st>>>(p, n_planes)
    if constexpr (ALLV) {
        if (neg1) {
            if (cp == 0) LAUNCH6(true, 0); else if (cp == 1) LAUNCH6(true, 1); else LAUNCH6(true, 2);
        } else {
            if (cp == 0) LAUNCH6(false, 0); else if (cp == 1) LAUNCH6(false, 1); else LAUNCH6(false, 2);
        }
    } else {
        LAUNCH6(true, 1);
    }
#undef LAUNCH6
    return check_launch("spmv_pattern_box6") == SPMVB_OK ? 0 : -1;
}

// v3 launch: returns 1 when the configuration / alignment is not served (caller falls back to v2)
template <int R, int WC, int Q, int LPS, int MINB, bool ALLV, int WA = 1>
static int launch_box3(const spmvb_matrix *a, PatternArgs &p, cudaStream_t st) {
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    const int n_planes = (int)((n_rows + sz - 1) / sz);
    const bool neg1 = p.v_off == -1.0;
    const int cp = a->box.center_pos;
    if (!ALLV && !(neg1 && cp == 1)) return 1;
    dim3 grid((p.sy + 64 * WA - 1) / (64 * WA), (p.plane_lines + R - 1) / R, (n_planes + (WC / WA) * Q - 1) / ((WC / WA) * Q));
    dim3 block(WC * 32);
#define LAUNCH3(NEG, CP) spmv_pattern_box3_kernel<R, WC, Q, LPS, MINB, NEG, CP, WA><<<grid, block, 0, st>>>(p, n_planes)
    if constexpr (ALLV) {
        if (neg1) {
            if (cp == 0) LAUNCH3(true, 0); else if (cp == 1) LAUNCH3(true, 1); else LAUNCH3(true, 2);
        } else {
            if (cp == 0) LAUNCH3(false, 0); else if (cp == 1) LAUNCH3(false, 1); else LAUNCH3(false, 2);
        }
    } else {
        LAUNCH3(true, 1);
    }
#undef LAUNCH3
    return check_launch("spmv_pattern_box3") == SPMVB_OK ? 0 : -1;
}

// v4 (shared-memory ring) launch: returns 1 when not served
template <int R, int WC, int Q, int DEPTH, int MINB>
static int launch_box5(const spmvb_matrix *a, PatternArgs &p, cudaStream_t st) {
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    const int n_planes = (int)((n_rows + sz - 1) / sz);
    if (!(p.v_off == -1.0 && a->box.center_pos == 1)) return 1;
    if (p.sy % 4 || (p.g0 + p.row_begin) % 4 || p.row_begin % 4) return 1;
    constexpr int NP = WC * Q;
    const size_t smem = (size_t)DEPTH * ((NP + 2) * 68 * 8 + NP * 64 * 4);
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(spmv_pattern_box5_kernel<R, WC, Q, DEPTH, MINB, true, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
        attr_set = true;
    }
    dim3 grid((p.sy + 63) / 64, (p.plane_lines + R - 1) / R, (n_planes + NP - 1) / NP);
    spmv_pattern_box5_kernel<R, WC, Q, DEPTH, MINB, true, 1><<<grid, WC * 32, smem, st>>>(p, n_planes);
    return check_launch("spmv_pattern_box5") == SPMVB_OK ? 0 : -1;
}

// pipelined ring launch: returns 1 when not served
template <int R, int WC, int Q, int DEPTH, int MINB>
static int launch_box7(const spmvb_matrix *a, PatternArgs &p, cudaStream_t st) {
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    const int n_planes = (int)((n_rows + sz - 1) / sz);
    if (!(p.v_off == -1.0 && a->box.center_pos == 1)) return 1;
    if (p.sy % 4 || (p.g0 + p.row_begin) % 4 || p.row_begin % 4) return 1;
    constexpr int NP = WC * Q;
    const size_t smem = (size_t)DEPTH * ((NP + 2) * 68 * 8 + NP * 64 * 4);
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(spmv_pattern_box7_kernel<R, WC, Q, DEPTH, MINB, true, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
        attr_set = true;
    }
    dim3 grid((p.sy + 63) / 64, (p.plane_lines + R - 1) / R, (n_planes + NP - 1) / NP);
    spmv_pattern_box7_kernel<R, WC, Q, DEPTH, MINB, true, 1><<<grid, WC * 32, smem, st>>>(p, n_planes);
    return check_launch("spmv_pattern_box7") == SPMVB_OK ? 0 : -1;
}

// warp-specialised TMA ring launch: returns 1 when not served
template <int R, int DEPTH, int WZ>
static int launch_box8(const spmvb_matrix *a, PatternArgs &p, cudaStream_t st) {
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    const int n_planes = (int)((n_rows + sz - 1) / sz);
    if (!(p.v_off == -1.0 && a->box.center_pos == 1)) return 1;
    if (p.sy % 4 || p.sy < 256 || (p.g0 + p.row_begin) % 4 || p.row_begin % 4 || (uintptr_t)p.ids % 16) return 1;
    constexpr int NP = 2 * WZ;
    constexpr size_t stage = (size_t)(NP + 2) * 260 * 8 + NP * 256 * 4;
    const size_t smem = stage * DEPTH;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(spmv_pattern_box8_kernel<R, DEPTH, WZ, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess) return -1;
        attr_set = true;
    }
    const int tx = (p.sy + 255) / 256, ty = (p.plane_lines + R - 1) / R, tz = (n_planes + NP - 1) / NP;
    const int grid = std::min(tx * ty * tz, 148);
    spmv_pattern_box8_kernel<R, DEPTH, WZ, true, 1><<<grid, (1 + 4 * WZ) * 32, smem, st>>>(p, n_planes, ty, tz, tx);
    return check_launch("spmv_pattern_box8") == SPMVB_OK ? 0 : -1;
}

// Conditions of the v3 kernel: vector loads need even strides/offsets and 16-byte aligned
// arrays; all in-tile offsets must fit 32 bits; masks must fit the shared-memory table.
static bool box3_ok(const spmvb_matrix *a, const PatternArgs &p) {
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    return (p.sy % 2 == 0) && ((p.g0 + p.row_begin) % 2 == 0) && (p.row_begin % 2 == 0) &&
           ((uintptr_t)p.x % 16 == 0) && ((uintptr_t)p.y % 16 == 0) && ((uintptr_t)p.ids % 8 == 0) &&
           a->n_patterns <= kDictSmemPat && 6 * sz + 128 * (int64_t)p.sy + 4096 < INT32_MAX;
}

static int launch_pattern(const spmvb_matrix *a, const double *x, int64_t x_col0, int64_t x_len, double *y,
                          int row_begin, int row_end, cudaStream_t st) {
    if (row_end > row_begin) {
        PatternArgs p;
        p.ids = static_cast<const int32_t *>(a->s[SPMVB_S_ROW_PATTERN]);
        p.x = x; p.y = y;
        p.g0 = a->row_offset - x_col0;
        p.x_len = x_len;
        p.disp_off = a->d_disp_off32;
        p.disp = static_cast<const int32_t *>(a->s[SPMVB_S_DISP_FLAT]);
        p.ends = static_cast<const int32_t *>(a->s[SPMVB_S_ENDS_FLAT]);
        p.table = static_cast<const double *>(a->s[SPMVB_S_TABLE]);
        p.masks = a->d_masks;
        p.n_patterns = a->n_patterns; p.m = a->m; p.disp_total = (int)a->disp_total;
        p.row_begin = row_begin; p.row_end = row_end;
        p.sy = a->box.sy; p.plane_lines = a->box.valid ? a->box.sz / a->box.sy : 0;
        p.v_off = a->box.valid ? a->h_table[a->box.k_off] : 0.0;
        p.v_center = a->box.valid ? a->h_table[a->box.k_center] : 0.0;
        const Options &o = options();
        p.prefetch = o.box_prefetch >= 0 ? o.box_prefetch : 2;
        p.prefetch_l1 = o.box_prefetch_l1;
        p.debug_nochain = o.debug_nochain;
        const bool use_box = a->box.valid && o.pattern_kernel != 1;
        if (o.pattern_kernel == 2 && !a->box.valid)
            return fail(SPMVB_ERR_INVALID_ARGUMENT, "box kernel requested but the dictionary has no box plan");
        if (use_box) {
            int rc3 = 1;  // 1 = not served by v3
            if (o.pattern_kernel != 3 && box3_ok(a, p)) {
                const int64_t n_planes = ((int64_t)row_end - row_begin + (int64_t)p.sy * p.plane_lines - 1) / ((int64_t)p.sy * p.plane_lines);
                if (n_planes == 1) rc3 = launch_box3<16, 4, 1, 2, 3, false>(a, p, st);  // single-plane ranges (slab boundary planes)
                else switch (o.box_march) {
                    // measured alternatives kept selectable for A/B (profiles/r01_probe256_*.log, 256^3):
                    case 1: rc3 = launch_box3<16, 4, 2, 1, 3, false>(a, p, st); break;      // R=16 tiles            124 us
                    case 5: rc3 = launch_box3<16, 4, 1, 2, 3, false>(a, p, st); break;      // 1 plane, 2 lines/step 116-121 us
                    case 12: rc3 = launch_box3<16, 4, 2, 1, 3, false, 4>(a, p, st); break;  // CTA spans full lines  124 us
                    case 20: rc3 = launch_box5<16, 4, 2, 4, 3>(a, p, st); break;            // cp.async ring         137 us
                    case 35: rc3 = launch_box6<4, 8, 4, 2, 2, false>(a, p, st); break;      // 4 columns per thread  127 us
                    case 30: rc3 = launch_box6<8, 8, 4, 1, 2, false>(a, p, st); break;      // 8 columns per thread  183 us
                    case 47: rc3 = launch_box7<16, 4, 2, 8, 2>(a, p, st); break;            // pipelined ring        141 us
                    case 62: rc3 = launch_box8<8, 10, 2>(a, p, st); break;                  // warp-specialised TMA ring 208 us (spills)
                    // default <R=8 lines, 4 warps, Q=2 planes/thread, 1 line/step, 3 CTAs/SM>: 118 us
                    default: rc3 = launch_box3<8, 4, 2, 1, 3, true>(a, p, st); break;
                }
                if (rc3 < 0) return SPMVB_ERR_CUDA;
            }
            if (rc3 == 1) {  // v2: any stride / alignment / value pattern
                if (o.box_march == 11) SPMVB_TRY((launch_box_rw<32, 8, 1, 1>(a, p, st)));
                else SPMVB_TRY((launch_box_rw<16, 8, 2, 0>(a, p, st)));
            }
        } else {
            const int threads = 256;
            const int blocks = (row_end - row_begin + threads - 1) / threads;
            const bool dict_smem = a->disp_total <= kDictSmemDisp && a->n_patterns <= kDictSmemPat && a->m <= kDictSmemTab;
            if (dict_smem) spmv_pattern_generic_kernel<true><<<blocks, threads, 0, st>>>(p);
            else spmv_pattern_generic_kernel<false><<<blocks, threads, 0, st>>>(p);
            SPMVB_TRY(check_launch("spmv_pattern_generic"));
        }
    }
    if (a->n_exc > 0 && row_end > row_begin) {
        // exception slots whose rows fall in [row_begin,row_end)
        const auto &er = a->h_exc_rows;
        const int e0 = (int)(std::lower_bound(er.begin(), er.end(), row_begin) - er.begin());
        const int e1 = (int)(std::lower_bound(er.begin(), er.end(), row_end) - er.begin());
        SPMVB_TRY(launch_ell(static_cast<const double *>(a->s[SPMVB_S_EXC_VALUES]),
                             static_cast<const int32_t *>(a->s[SPMVB_S_EXC_COLUMNS]), a->w_exc, x, x_col0, y, e0, e1,
                             static_cast<const int32_t *>(a->s[SPMVB_S_EXC_ROWS]), st));
    }
    return SPMVB_OK;
}

}  // namespace spmvb

using namespace spmvb;

extern "C" {

int spmvb_spmv(const spmvb_matrix *a, const double *x_dev, int64_t x_col0, int64_t x_len, double *y_dev,
               int32_t row_begin, int32_t row_end, void *stream) {
    if (!a || !x_dev || !y_dev) return fail(SPMVB_ERR_INVALID_ARGUMENT, "spmv: NULL argument");
    if (row_begin < 0 || row_end > a->n || row_begin > row_end)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "spmv: row range [%d,%d) outside [0,%d)", row_begin, row_end, a->n);
    cudaStream_t st = as_stream(stream);
    switch (a->format) {
        case SPMVB_FMT_ELL:
            return launch_ell(static_cast<const double *>(a->s[SPMVB_S_VALUES]),
                              static_cast<const int32_t *>(a->s[SPMVB_S_COLUMNS]), a->width, x_dev, x_col0, y_dev,
                              row_begin, row_end, nullptr, st);
        case SPMVB_FMT_VT:
            return launch_vt(a, x_dev, x_col0, y_dev, row_begin, row_end, st);
        case SPMVB_FMT_PATTERN:
            return launch_pattern(a, x_dev, x_col0, x_len, y_dev, row_begin, row_end, st);
        default:
            return fail(SPMVB_ERR_INVALID_ARGUMENT, "spmv: format %d has no SpMV kernel", a->format);
    }
}

int spmvb_spmv_host(const spmvb_matrix *a, const double *x_host, int64_t x_len, double *y_host) {
    if (!a || !x_host || !y_host) return fail(SPMVB_ERR_INVALID_ARGUMENT, "spmv_host: NULL argument");
    if (a->row_offset != 0) return fail(SPMVB_ERR_INVALID_ARGUMENT, "spmv_host: handle is a slab (row_offset != 0)");
    if (x_len != a->n)  // SPEC.md:212,222,232 "length mismatch"
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "spmv: x has %lld entries, matrix has %d rows", (long long)x_len, a->n);
    // persistent device scratch: the matrix stays resident, only x and y cross the bus
    if (a->scratch_x_len < x_len || !a->scratch_x) {
        if (a->scratch_x) cudaFree(a->scratch_x);
        if (a->scratch_y) cudaFree(a->scratch_y);
        a->scratch_x = a->scratch_y = nullptr;
        a->scratch_x_len = 0;
        SPMVB_TRY(spmvb_vec_alloc(x_len, &a->scratch_x));
        SPMVB_TRY(spmvb_vec_alloc(a->n, &a->scratch_y));
        a->scratch_x_len = x_len;
    }
    SPMVB_CUDA(cudaMemcpyAsync(a->scratch_x, x_host, (size_t)x_len * 8, cudaMemcpyHostToDevice, nullptr));
    SPMVB_TRY(spmvb_spmv(a, a->scratch_x, 0, x_len, a->scratch_y, 0, a->n, nullptr));
    SPMVB_CUDA(cudaMemcpyAsync(y_host, a->scratch_y, (size_t)a->n * 8, cudaMemcpyDeviceToHost, nullptr));
    SPMVB_CUDA(cudaStreamSynchronize(nullptr));
    return SPMVB_OK;
}

}  // extern "C"
