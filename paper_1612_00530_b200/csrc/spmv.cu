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
    const double *v = sv + threadIdx.x * width;
    const int32_t *c = sc + threadIdx.x * width;
    double acc = 0.0;
#pragma unroll 9
    for (int k = 0; k < width; k++) acc = __dadd_rn(acc, __dmul_rn(v[k], __ldg(x + ((int64_t)c[k] - x_col0))));
    y[row_map ? row_map[r] : r] = acc;
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
    const int32_t *c = sc + threadIdx.x * width;
    const int32_t *e = se + threadIdx.x * m;
    double acc = 0.0;
    int idx = 0;
    for (int k = 0; k < m; k++) {
        double sum = 0.0;
        const int end = e[k];
        for (; idx < end; idx++) sum = __dadd_rn(sum, __ldg(x + ((int64_t)c[idx] - x_col0)));
        acc = __dadd_rn(acc, __dmul_rn(st[k], sum));
    }
    y[r] = acc;
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
        p.prefetch = o.box_prefetch >= 0 ? o.box_prefetch : 6;
        const bool use_box = a->box.valid && o.pattern_kernel != 1;
        if (o.pattern_kernel == 2 && !a->box.valid)
            return fail(SPMVB_ERR_INVALID_ARGUMENT, "box kernel requested but the dictionary has no box plan");
        if (use_box) {
            switch (o.box_march) {  // <R lines, WC warps, Q planes/thread, look-ahead>
                case 1: SPMVB_TRY((launch_box_rw<32, 8, 1, 1>(a, p, st))); break;
                case 2: SPMVB_TRY((launch_box_rw<32, 4, 2, 1>(a, p, st))); break;
                case 3: SPMVB_TRY((launch_box_rw<16, 4, 2, 1>(a, p, st))); break;
                case 4: SPMVB_TRY((launch_box_rw<32, 4, 2, 0>(a, p, st))); break;
                case 5: SPMVB_TRY((launch_box_rw<16, 4, 3, 0>(a, p, st))); break;
                case 6: SPMVB_TRY((launch_box_rw<32, 4, 4, 0>(a, p, st))); break;
                case 7: SPMVB_TRY((launch_box_rw<16, 4, 4, 0>(a, p, st))); break;
                case 8: SPMVB_TRY((launch_box_rw<16, 2, 4, 0>(a, p, st))); break;
                case 9: SPMVB_TRY((launch_box_rw<16, 8, 2, 0>(a, p, st))); break;
                default: SPMVB_TRY((launch_box_rw<32, 4, 2, 1>(a, p, st))); break;
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
