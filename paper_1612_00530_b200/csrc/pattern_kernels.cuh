// Pattern-format SpMV kernels shared by spmv_pattern.cu (production paths) and
// spmv_pattern_lab.cu (measured experiments): List 1 as written, the one-column
// sliding-window kernel (v2) and the default two-column kernel (box3).
//
// Arithmetic contract: every product and every sum is rounded
// separately (__dmul_rn / __dadd_rn, never contracted to FMA), in the reference's documented
// per-format order (inc/kernels.hpp:19-22), so results are bit-identical to the reference's
// `y[i] += a_ij * x_j` built for baseline x86-64.  Multiplication by -1.0 is exact, so
// `acc + (-1.0 * x)` is issued as `acc - x`.
#pragma once
#include "common.cuh"
#include "device_utils.cuh"

namespace spmvb {

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
    int64_t ids_avail;         // rows of the id stream from row_begin to its end (prefetch-reach guard)
    // box plan
    int sy, plane_lines;       // sy = stride of dy; plane_lines = sz / sy
    double v_off, v_center;
    int prefetch;              // L2 prefetch distance in lines
    int prefetch_l1;           // L1 prefetch distance in lines (v3), 0 = off
    int debug_nochain;         // measurement only: skip the FP64 chains (y = centre operand)
    int center_pos = 1;        // where the centre term sits in the summation order: 0 first, 1 last, 2 in place (BoxPlan)
    double *dot_partial = nullptr;  // fused x.y (CG's p.Ap): one partial sum per warp of the tensor-ring kernel, else nullptr
    int dot_capacity = 0;
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

static __device__ __noinline__ double pattern_row_cold(const PatternArgs &p, int id, int64_t xi) {
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
    const int cpos = CENTER_POS >= 0 ? CENTER_POS : p.center_pos;  // CENTER_POS = -1: read at run time (the general variant)
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
                    if (cpos == 0) {
#pragma unroll
                        for (int q = 0; q < Q; q++) acc[q] = __dadd_rn(acc[q], __dmul_rn(vc, w[sl[1]][q + 1][1]));
                    }
#pragma unroll
                    for (int t = 0; t < 27; t++) {
                        if (t == 13 && cpos != 2) continue;
                        const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            const double e = w[sl[dy]][q + dz][dx];
                            acc[q] = OFF_NEG1 ? __dsub_rn(acc[q], e) : __dadd_rn(acc[q], __dmul_rn(vo, e));
                        }
                    }
                    if (cpos == 1) {
#pragma unroll
                        for (int q = 0; q < Q; q++) acc[q] = __dadd_rn(acc[q], __dmul_rn(vc, w[sl[1]][q + 1][1]));
                    }
                } else {
                    // Masked rows: an absent entry contributes +0.0.  acc starts at +0.0 and can
                    // never become -0.0 (round to nearest), so adding +-0.0 leaves it unchanged
                    // bit for bit: identical to skipping the term as the reference does.
                    if (cpos == 0) {
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            const double pr = __dmul_rn(vc, w[sl[1]][q + 1][1]);
                            acc[q] = __dadd_rn(acc[q], (mk[q] >> 13 & 1u) ? pr : 0.0);
                        }
                    }
#pragma unroll
                    for (int t = 0; t < 27; t++) {
                        if (t == 13 && cpos != 2) continue;
                        const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            const double e = w[sl[dy]][q + dz][dx];
                            const bool on = mk[q] >> t & 1u;
                            if (OFF_NEG1) acc[q] = __dsub_rn(acc[q], on ? e : 0.0);
                            else acc[q] = __dadd_rn(acc[q], on ? __dmul_rn(vo, e) : 0.0);
                        }
                    }
                    if (cpos == 1) {
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
                                           double (&acc)[LPS][Q][2], int cp_rt) {
    const int cpos = CENTER_POS >= 0 ? CENTER_POS : cp_rt;
    // MODE 0: operands straight from the window (with SELL/SELR: halo operands zeroed per lane)
    // MODE 1: every operand selected by its mask bit
    // line l of the step reads slots (kb+l-1, kb+l, kb+l+1) mod S for dy = -1, 0, +1
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
    if (cpos == 0) centre();
#pragma unroll
    for (int t = 0; t < 27; t++) {
        if (t == 13 && cpos != 2) continue;
        const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
#pragma unroll
        for (int l = 0; l < LPS; l++)
#pragma unroll
            for (int q = 0; q < Q; q++)
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    double e = w[(kb + l + dy + S - 1) % S][q + dz][i + dx];
                    if (MODE == 0 && SELL && i + dx == 0) e = zl[l][q] ? 0.0 : e;
                    if (MODE == 0 && SELR && i + dx == 3) e = zr[l][q] ? 0.0 : e;
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
    if (cpos == 1) centre();
}

// Row classes (shared-memory tables indexed by pattern id + 1; entry 0 serves exception
// rows, id = -1, which are computed as full rows and never stored).  cls0 is for rows in
// the thread's left column, cls1 for its right column:
//   0 full box; 1 (cls0) only the nine dx=-1 entries missing; 2 (cls1) only the nine
//   dx=+1 entries missing; 4 any other mask (fully masked chain / List 1).
struct Box3Smem {
    uint32_t cls0, cls1, masks;  // 32-bit shared addresses of the three tables
};

template <int Q, int LPS, bool OFF_NEG1, int CENTER_POS, int LA = 0>
__device__ __forceinline__ void box3_march(const PatternArgs &p, const Box3Smem sm, const double *__restrict__ xw,
                                           const int32_t *__restrict__ idw, double *__restrict__ yw, int64_t xi_w, int lane,
                                           int nb, bool lane_ok, int nq) {
    // window slots: lines jb-1 .. jb+LPS in use by the step, plus LA steps of look-ahead in flight
    constexpr int S = LPS * (1 + LA) + 2, P = Q + 2;
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
#pragma unroll
    for (int l = 0; l <= LA * LPS; l++) load_line(l, l * sy);
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
                for (int l = 0; l < LPS; l++) load_line((kb + 1 + l + LA * LPS) % S, (1 + l + LA * LPS) * sy);
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
                    box3_chain<Q, S, LPS, OFF_NEG1, CENTER_POS, 0, false, false>(w, kb, mk, zl, zr, vc, vo, acc, p.center_pos);
                } else if (vote == 1 || vote == 2) {
#pragma unroll
                    for (int l = 0; l < LPS; l++)
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            zl[l][q] = c0[l][q] != 0;
                            zr[l][q] = c1[l][q] != 0;
                        }
                    if (vote == 1) box3_chain<Q, S, LPS, OFF_NEG1, CENTER_POS, 0, true, false>(w, kb, mk, zl, zr, vc, vo, acc, p.center_pos);
                    else box3_chain<Q, S, LPS, OFF_NEG1, CENTER_POS, 0, false, true>(w, kb, mk, zl, zr, vc, vo, acc, p.center_pos);
                } else {
#pragma unroll
                    for (int l = 0; l < LPS; l++)
#pragma unroll
                        for (int q = 0; q < Q; q++)
#pragma unroll
                            for (int i = 0; i < 2; i++) mk[l][q][i] = lds_u32(sm.masks + 4 + 4 * id[l][q][i]);
                    box3_chain<Q, S, LPS, OFF_NEG1, CENTER_POS, 1, false, false>(w, kb, mk, zl, zr, vc, vo, acc, p.center_pos);
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

template <int R, int WC, int Q, int LPS, int MINB, bool OFF_NEG1, int CENTER_POS, int WA = 1, int LA = 0>
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
    const int64_t x_hi = xi_w + 64 + (int64_t)(nb_up + LPS * (1 + LA) + pf) * sy + (int64_t)Q * sz + 1;
    const int64_t id_hi = r_w + 64 + (int64_t)(nb_up + LPS + pf) * sy + (int64_t)(nq - 1) * sz;  // ids prefetch reach
    const bool interior = last_row < n_rows && x_lo >= 0 && x_hi < p.x_len && id_hi <= p.ids_avail + 1024;
    if (interior) {
        box3_march<Q, LPS, OFF_NEG1, CENTER_POS, LA>(p, sm, p.x + xi_w, p.ids + p.row_begin + r_w, p.y + p.row_begin + r_w, xi_w,
                                                 lane, nb, lane * 2 + 1 < cols_ok, nq);
    } else {
        box3_edge_tile<Q, OFF_NEG1, CENTER_POS>(p, s_masks, r_w, lane, nb, n_rows, nq, cols_ok);
    }
}


}  // namespace spmvb
