// Measured experiments on the pattern-format SpMV: shared-memory rings
// (cp.async and TMA bulk copies), wide tiles, software pipelining, warp specialisation.  None of
// them beats the default box3 kernel yet; they stay selectable (option "box_march") so the
// numbers in profiles/ can be reproduced, and they are covered by the same parity tests.
#include <algorithm>

#include "pattern_kernels.cuh"
#include "spmv_internal.cuh"

namespace spmvb {

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
                    if (vote == 0) box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, false, false>(w, k, mk, zl, zr, vc, vo, acc, CENTER_POS);
                    else if (vote == 1) box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, true, false>(w, k, mk, zl, zr, vc, vo, acc, CENTER_POS);
                    else if (vote == 2) box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, false, true>(w, k, mk, zl, zr, vc, vo, acc, CENTER_POS);
                    else {
                        box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 1, false, false>(w, k, mk, zl, zr, vc, vo, acc, CENTER_POS);
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
    const bool interior = last_row < n_rows && x_lo >= 0 && x_hi < p.x_len && id_hi <= p.ids_avail + 1024;
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
                    box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, true, true>(w, k, mk, zl1, zr1, vc, vo, acc, CENTER_POS);  // ... under chain j
                } else {
                    load_line((k + 2) % S, j + 2);
                    other_n = classify(j + 1, idn, zln, zrn);
#pragma unroll
                    for (int q = 0; q < Q; q++)
#pragma unroll
                        for (int i = 0; i < 2; i++) mk[0][q][i] = lds_u32(mask_a + 4 + 4 * id[q][i]);
                    box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 1, false, false>(w, k, mk, zl1, zr1, vc, vo, acc, CENTER_POS);
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
                            box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, false, false>(w, k, mk, zl, zr, vc, vo, acc, CENTER_POS);
                        } else if (vote == 1 || vote == 2) {
#pragma unroll
                            for (int q = 0; q < Q; q++) { zl[0][q] = c0v[q] != 0; zr[0][q] = c1v[q] != 0; }
                            if (vote == 1) box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, true, false>(w, k, mk, zl, zr, vc, vo, acc, CENTER_POS);
                            else box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 0, false, true>(w, k, mk, zl, zr, vc, vo, acc, CENTER_POS);
                        } else {
#pragma unroll
                            for (int q = 0; q < Q; q++)
#pragma unroll
                                for (int i = 0; i < 2; i++) mk[0][q][i] = lds_u32(sm.masks + 4 + 4 * id[0][q][i]);
                            box3_chain<Q, S, 1, OFF_NEG1, CENTER_POS, 1, false, false>(w, k, mk, zl, zr, vc, vo, acc, CENTER_POS);
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
    static PerDevice<bool> attr_set;
    if (!attr_set.get()) {
        if (cudaFuncSetAttribute(spmv_pattern_box5_kernel<R, WC, Q, DEPTH, MINB, true, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
        attr_set.get() = true;
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
    static PerDevice<bool> attr_set;
    if (!attr_set.get()) {
        if (cudaFuncSetAttribute(spmv_pattern_box7_kernel<R, WC, Q, DEPTH, MINB, true, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
        attr_set.get() = true;
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
    static PerDevice<bool> attr_set;
    if (!attr_set.get()) {
        if (cudaFuncSetAttribute(spmv_pattern_box8_kernel<R, DEPTH, WZ, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess) return -1;
        attr_set.get() = true;
    }
    const int tx = (p.sy + 255) / 256, ty = (p.plane_lines + R - 1) / R, tz = (n_planes + NP - 1) / NP;
    const int grid = std::min(tx * ty * tz, 148);
    spmv_pattern_box8_kernel<R, DEPTH, WZ, true, 1><<<grid, (1 + 4 * WZ) * 32, smem, st>>>(p, n_planes, ty, tz, tx);
    return check_launch("spmv_pattern_box8") == SPMVB_OK ? 0 : -1;
}

int launch_pattern_lab(int which, const spmvb_matrix *a, PatternArgs &p, cudaStream_t st) {
    if (a->n_patterns > kDictSmemPat) return 1;
    switch (which) {  // times: 256^3 on one B200 (profiles/r01_probe256_*.log); box3 default = 118 us
        case 20: return launch_box5<16, 4, 2, 4, 3>(a, p, st);       // cp.async ring                  137 us
        case 35: return launch_box6<4, 8, 4, 2, 2, false>(a, p, st); // 4 columns per thread           127 us
        case 30: return launch_box6<8, 8, 4, 1, 2, false>(a, p, st); // 8 columns per thread           183 us
        case 47: return launch_box7<16, 4, 2, 8, 2>(a, p, st);       // software-pipelined ring        141 us
        case 62: return launch_box8<8, 10, 2>(a, p, st);             // warp-specialised TMA ring      208 us (spills)
        default: return 1;
    }
}

}  // namespace spmvb
