// Pattern-format SpMV (inc/compress.hpp:48-76; inc/kernels.hpp:25,35-36; PAPER.md:797-813 List 1):
// the "tensor ring" kernel, the default for ranges of at least 8 planes.  x is viewed through a 3-D
// TMA tensor map [plane][line][column] whose strides (sz, sy, 1) come from the dictionary's box plan;
// every warp owns a 64-column strip of Q planes and marches over lines.  One elected lane fetches the
// next line set -- 68 columns x (Q+2) planes of x and, through a second int32 view, the 72 x Q pattern
// ids of that line, one cp.async.bulk.tensor each -- into the warp's private shared-memory ring
// (completion on an mbarrier), and all lanes take the 27 operands of their rows from shared memory with
// 128-bit loads.  No register window and no per-thread global loads.  DESIGN.md section 6 has the
// measurements, the ablations and the dead ends.
//
// Alignment.  A TMA box must start on a 16-byte boundary, i.e. at an even column, and a thread wants
// its four operands (columns a-1 .. a+2 for its rows a, a+1) as two aligned 128-bit shared loads.
// Both hold when a is odd: strip s covers columns 64s-1 .. 64s+62 and its box starts at 64s-2.
// Column -1 of strip 0 is a dummy; the columns past the last strip (one column when 64 | sy) are
// summed row by row from global memory after the marches.
//
// Exactness.  Elements outside the tensor view are zero-filled by the TMA unit.  A row whose
// dictionary mask is exactly "the full box minus the entries that fall outside the view" is
// therefore served by the plain 27-term chain: absent operands are +0.0 and leave the accumulator
// unchanged bit for bit (it can never be -0.0).  That is every row of a stencil matrix whose x view
// is aligned with the grid.  A row whose entries are another sub-box inside the view is summed again
// with every operand selected by its mask bit; any other row (another dictionary pattern, entries
// outside the view, a view that is not aligned with the grid) is recomputed by List 1 as written, so
// the result is always the reference's order.  Exception rows (id -1) are left to the exception
// block, as in the other kernels.
#include <cuda.h>  // CUtensorMap and enums only; the encoder is resolved through the runtime (no -lcuda)

#include <algorithm>

#include "pattern_kernels.cuh"
#include "spmv_internal.cuh"

namespace spmvb {

constexpr uint32_t kDyLoBits = 0x01C0E07u;  // box entries with dy = -1
constexpr uint32_t kDyHiBits = kDyLoBits << 6;
constexpr uint32_t kDzLoBits = 0x1FFu;  // dz = -1
constexpr uint32_t kDzHiBits = 0x1FFu << 18;
constexpr int kStripCols = 64;            // columns per warp
constexpr int kBoxCols = kStripCols + 4;  // columns 64s-2 .. 64s+65 (the first and last are alignment padding)
constexpr int kRingWarps = 4;
#ifndef RING_LEFT_MODE
#define RING_LEFT_MODE 1  // 1: the left-over column's rows are summed by the whole CTA at the end of a march (chunk-per-CTA kernels); 0: per step
#endif

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *tm, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
// TMA-engine prefetch of the same box into L2 only
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap *tm, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(tm), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory"); }
__device__ __forceinline__ void sts_f64x2(uint32_t addr, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1,%2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}

constexpr int kIdBoxCols = kStripCols + 8;  // id box: columns 64s-4 .. 64s+67 (a 16-byte aligned start for 4-byte ids)

template <int Q, int S, bool IDT, int LPS = 1>
struct RingLayout {
    static constexpr int P = Q + 2;
    static constexpr uint32_t kLineBytes = kBoxCols * 8;                    // one plane of a line set of x
    static constexpr uint32_t kXBytes = (P * kLineBytes + 127u) / 128u * 128u;  // TMA destinations are 128-byte aligned
    static constexpr uint32_t kIdLineBytes = kIdBoxCols * 4;
    static constexpr uint32_t kIdBytes = IDT ? Q * kIdLineBytes : 0;        // the ids of the set's line ride along
    static constexpr uint32_t kSetBytes = P * kLineBytes + kIdBytes;        // bytes the TMA boxes of one set deliver
    static constexpr uint32_t kSlotBytes = kXBytes + (kIdBytes + 127u) / 128u * 128u;
    static constexpr uint32_t kRingBytes = kRingWarps * S * kSlotBytes;
    static constexpr uint32_t kBarBytes = kRingWarps * S * 8;
    static constexpr uint32_t kMaskBytes = ((kDictSmemPat + 1) * 4 + 15u) / 16u * 16u;  // one private copy of the mask table per warp
    static constexpr uint32_t kBase = kRingBytes + kBarBytes + kRingWarps * kMaskBytes;
    // Side buffer of the left-over column (chunk-per-CTA kernels, see the kernel): columns sy-2, sy-1 of the lines b0-1 .. b0+nb of a
    // march, every plane of the set, 16 bytes each, and the nb x Q pattern ids of column sy-1.  A march is at most kLeftCap lines.
    static constexpr int kLeftCap = Q >= 6 ? 46 : LPS == 2 ? 28 : 16;
    static constexpr uint32_t kLeftXBytes = (kLeftCap + 2) * P * 16;
    static constexpr uint32_t kLeftBytes = (kLeftXBytes + kLeftCap * Q * 4 + 15u) / 16u * 16u;
    static constexpr uint32_t kTotal = kBase + 128;  // + alignment slack
};

// Rare path of the direct variant, kept out of line so that its registers do not weigh on the main loop: the sums
// of one step again, every operand selected by its row's own 27-bit mask (absent entries contribute +0.0), operands
// re-read from the three line slots of the ring; the rows stay interleaved as in the main chain.
template <int Q, bool OFF_NEG1, int CENTER_POS, uint32_t LINE_BYTES>
__device__ __noinline__ void ring_masked_step(uint32_t sl0, uint32_t sl1, uint32_t sl2, const uint32_t *mk, double vc, double vo,
                                              double *out, int cp_rt) {
    constexpr int P = Q + 2;
    const int cpos = CENTER_POS >= 0 ? CENTER_POS : cp_rt;
    const uint32_t sl[3] = {sl0, sl1, sl2};
    double acc[Q][2], xc[Q][2];
#pragma unroll
    for (int q = 0; q < Q; q++) {
        const double2 u = lds_f64x2(sl[1] + (q + 1) * LINE_BYTES), v = lds_f64x2(sl[1] + (q + 1) * LINE_BYTES + 16);
        xc[q][0] = (mk[q * 2] >> 13 & 1u) ? __dmul_rn(vc, u.y) : 0.0;
        xc[q][1] = (mk[q * 2 + 1] >> 13 & 1u) ? __dmul_rn(vc, v.x) : 0.0;
        acc[q][0] = acc[q][1] = 0.0;
        if (cpos == 0) acc[q][0] = __dadd_rn(acc[q][0], xc[q][0]), acc[q][1] = __dadd_rn(acc[q][1], xc[q][1]);
    }
#pragma unroll
    for (int pz = 0; pz < P; pz++)
#pragma unroll
        for (int dy = 0; dy < 3; dy++) {
            const double2 u = lds_f64x2(sl[dy] + pz * LINE_BYTES), v = lds_f64x2(sl[dy] + pz * LINE_BYTES + 16);
            const double e[4] = {u.x, u.y, v.x, v.y};
#pragma unroll
            for (int dx = 0; dx < 3; dx++)
#pragma unroll
                for (int q = 0; q < Q; q++) {
                    const int dz = pz - q;
                    if (dz < 0 || dz > 2) continue;
                    const int t = dz * 9 + dy * 3 + dx;
#pragma unroll
                    for (int i = 0; i < 2; i++) {
                        const bool on = mk[q * 2 + i] >> t & 1u;
                        if (t == 13) {
                            if (cpos == 2) acc[q][i] = __dadd_rn(acc[q][i], xc[q][i]);
                        } else if (OFF_NEG1) {
                            acc[q][i] = __dsub_rn(acc[q][i], on ? e[i + dx] : 0.0);
                        } else {
                            acc[q][i] = __dadd_rn(acc[q][i], on ? __dmul_rn(vo, e[i + dx]) : 0.0);
                        }
                    }
                }
        }
#pragma unroll
    for (int q = 0; q < Q; q++)
#pragma unroll
        for (int i = 0; i < 2; i++) out[q * 2 + i] = cpos == 1 ? __dadd_rn(acc[q][i], xc[q][i]) : acc[q][i];
}

// -----------------------------------------------------------------------------------------
// The kernel.  One wave of persistent CTAs; the (strip or strip group, plane group) columns of the view, pl lines each,
// form one sequence of line steps.  Two schedules (see launch_pattern_ring): equal contiguous chunks of that sequence,
// one per CTA (its four warps on the four strips of the same lines) or per warp; or tiles of a few lines dealt out
// round-robin.  A chunk that crosses a column end (or the rotation point of its column) is two marches.  The ring
// (slot = set number mod S, parity from the set number) runs on across marches.  The rows of the left-over columns are
// dealt out to the warps and summed after their marches.
// -----------------------------------------------------------------------------------------
// One row of a left-over column.  The id and all in-view box operands are requested together (one memory latency);
// the row's mask then decides whether the plain sum is exact (same rule as the strips) or List 1 runs as written.
// Returns y[row] * x[row's own column] (0 when there is no such row): the fused dot of the DOT instantiation.
template <bool OFF_NEG1, int CENTER_POS>
__device__ __forceinline__ double ring_leftover_row(const PatternArgs &p, uint32_t s_masks, int col, int line, int c, int np_x) {
    const int sy = p.sy, pl = p.plane_lines;
    const int cpos = CENTER_POS >= 0 ? CENTER_POS : p.center_pos;
    const int64_t sz = (int64_t)sy * pl;
    const int64_t xi = col + (int64_t)sy * line + sz * c;
    const int64_t row = xi - p.g0;
    if (row < p.row_begin || row >= p.row_end) return 0.0;
    const uint32_t oob = (col == 0 ? kLBits : 0u) | (col == sy - 1 ? kRBits : 0u) | (line == 0 ? kDyLoBits : 0u) |
                         (line == pl - 1 ? kDyHiBits : 0u) | (c == 0 ? kDzLoBits : 0u) | (c == np_x - 1 ? kDzHiBits : 0u);
    const uint32_t in_view = c < np_x ? (kFullBox & ~oob) : 0u;
    const int id = __ldg(p.ids + row);
    double xv[27];
#pragma unroll
    for (int e = 0; e < 27; e++)
        xv[e] = (in_view >> e & 1u) ? __ldg(p.x + (xi + (e % 3 - 1) + (int64_t)sy * ((e / 3) % 3 - 1) + sz * (e / 9 - 1))) : 0.0;
    if (id < 0) return 0.0;
    if (in_view != 0 && lds_u32(s_masks + 4 + 4 * id) == in_view) {
        double acc = 0.0;
        if (cpos == 0) acc = __dadd_rn(acc, __dmul_rn(p.v_center, xv[13]));
#pragma unroll
        for (int e = 0; e < 27; e++) {
            if (e == 13) {
                if (cpos == 2) acc = __dadd_rn(acc, __dmul_rn(p.v_center, xv[13]));
            } else if (OFF_NEG1) {
                acc = __dsub_rn(acc, xv[e]);
            } else {
                acc = __dadd_rn(acc, __dmul_rn(p.v_off, xv[e]));
            }
        }
        if (cpos == 1) acc = __dadd_rn(acc, __dmul_rn(p.v_center, xv[13]));
        p.y[row] = acc;
        return __dmul_rn(acc, xv[13]);
    } else {
        const double acc = pattern_row(p, p.disp, p.ends, p.table, id, xi);
        p.y[row] = acc;
        return in_view != 0 ? __dmul_rn(acc, __ldg(p.x + xi)) : 0.0;
    }
}

template <int Q, int S, int MINB, bool OFF_NEG1, int CENTER_POS, bool IDT, int PFD = 0, int DBG = 0, bool CTAC = false, bool DOT = false, int LPS = 1>
__global__ void __launch_bounds__(kRingWarps * 32, MINB)
    spmv_pattern_ringp_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm_ids, PatternArgs p, int c_lo,
                              int c_hi, int np_x, int n_strips, int left_lo, int left_in_ring, int id_plane0, int total_steps, int steps_per_warp,
                              int steps_rem, int tile_lines, int rot) {
    using L = RingLayout<Q, S, IDT, LPS>;
    constexpr int P = L::P;
    static_assert(LPS == 1 || (LPS == 2 && IDT && CTAC && DBG == 0 && PFD == 0 && S >= 6), "two lines per step: chunk-per-CTA kernels with the ids in the ring");
    const int cpos = CENTER_POS >= 0 ? CENTER_POS : p.center_pos;  // CENTER_POS = -1: the general variant reads it at run time
    extern __shared__ unsigned char smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 127u) & ~127u;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sy = p.sy, pl = p.plane_lines;
    const int sz = sy * pl;
    const int rb = p.row_begin;
    const unsigned n_range = (unsigned)(p.row_end - p.row_begin);
    const uint32_t ring = sbase + warp * (S * L::kSlotBytes);
    const uint32_t bars = sbase + L::kRingBytes + warp * (S * 8);
    const uint32_t s_masks = sbase + L::kRingBytes + L::kBarBytes + warp * L::kMaskBytes;  // this warp's copy; entry 0 serves id = -1
    // left_in_ring == 2: the rows of the left-over column are summed by the whole CTA at the end of each march, from a side buffer
    // that every thread helps to fill (cp.async) when the march begins -- nothing per step, no extra work on the last strip's warp
    constexpr bool LFLUSH = RING_LEFT_MODE == 1 && IDT && DBG == 0 && CTAC;
    const uint32_t s_left = sbase + L::kBase;
    // PDL: the next launch of the stream may take this CTA's place as soon as it exits; this launch, in turn, may have been
    // started while the kernel before it was still draining -- no global memory is touched before the wait below.
    pdl_launch_dependents();
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < S; s++) mbar_init(bars + 8 * s, 1);
        fence_mbar_init();
    }
    if (threadIdx.x == 0) {  // the descriptors live in the kernel parameters: fetched ahead of their first use
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tm) : "memory");
        if (IDT) asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_ids) : "memory");
    }
    __syncwarp();  // this warp's barriers are initialised; no other warp ever touches them
    pdl_grid_dependency_wait();
    bool masks_staged = false;  // the mask table is staged behind the first line sets' fetches; no CTA barrier anywhere

    const int gw = blockIdx.x * kRingWarps + warp, n_warps = gridDim.x * kRingWarps;
    const int n_sg = (n_strips + kRingWarps - 1) / kRingWarps;  // CTAC: columns are (group of 4 strips, plane group)
    const int32_t *__restrict__ ids = p.ids;
    double *__restrict__ y = p.y;
    const double vc = p.v_center, vo = p.v_off;
    const uint32_t lane_off = lane * 16;
    uint32_t gs = 0;  // sets issued so far by this warp: slot = set number % S, parity = (set number / S) & 1
    double dsum = 0.0;  // DOT: this thread's share of x.y, rows in schedule order
    // CTAC: a work unit belongs to the CTA and its four warps take the four strips of the same lines (they then read
    // whole contiguous lines of x together); otherwise every warp has units of its own.
    // tile_lines == 0: one contiguous chunk of the column-major step sequence per unit (steps_per_warp steps);
    // tile_lines  > 0: tiles of that many lines, columns fastest, dealt out round-robin -- the tiles in flight then
    //                  stay within a few plane groups of each other (halo planes are re-read from L2).
    const int me = CTAC ? (int)blockIdx.x : gw, n_me = CTAC ? (int)gridDim.x : n_warps;
    const int n_cols = (CTAC ? n_sg : n_strips) * ((c_hi - c_lo + Q) / Q);
    const int n_tiles = tile_lines > 0 ? n_cols * ((pl + tile_lines - 1) / tile_lines) : 0;
    int tile = me;
    // unit `me` takes steps_per_warp steps, the first steps_rem units one more: every unit of a full wave has work
    int s_pos = me * steps_per_warp + min(me, steps_rem);
    const int s_end = min(total_steps, s_pos + steps_per_warp + (me < steps_rem ? 1 : 0));
#pragma unroll 1
    while (true) {
        int col_idx, b0, nb;
        if (tile_lines > 0) {
            if (tile >= n_tiles) break;
            col_idx = tile % n_cols;
            b0 = (tile / n_cols) * tile_lines;
            nb = min(tile_lines, pl - b0);
            tile += n_me;
        } else {
            if (s_pos >= s_end) break;
            col_idx = s_pos / pl;
            const int u = s_pos - col_idx * pl;  // position in the column's line sequence
            // The line sequence of plane group g starts at line g*rot (cyclically).  rot = (steps per plane group) - k * (chunk
            // length) for the nearest k: the CTA k chunks further on works on the next plane group and is then on the same lines
            // at the same time, so the halo planes the two groups share are read from DRAM once.
            b0 = (int)((u + (int64_t)(col_idx / (CTAC ? n_sg : n_strips)) * rot) % pl);
            nb = min(min(pl - u, pl - b0), s_end - s_pos);
            if (LFLUSH && left_in_ring == 2) nb = min(nb, L::kLeftCap);  // what the side buffer holds (the chunk goes on with another march)
            s_pos += nb;
        }
        const int strip = CTAC ? (col_idx % n_sg) * kRingWarps + warp : col_idx % n_strips;
        const int c0 = c_lo + (col_idx / (CTAC ? n_sg : n_strips)) * Q;
        const bool cta_left = LFLUSH && left_in_ring == 2 && (col_idx % n_sg) == n_sg - 1;  // this CTA's strips end at column sy-2
        if (!(CTAC && strip >= n_strips)) {  // (else: no such strip in this group)
        const int a_w = strip * kStripCols - 1;  // first column of the strip (odd; -1 for strip 0)
        const int n_sets = nb + 2;               // line sets b0-1 .. b0+nb
        auto issue = [&](int k) {  // elected lane: line set k of this march -> slot (gs + k) % S
            const uint32_t slot = (gs + k) % S, bar = bars + 8 * slot;
            mbar_expect_tx(bar, L::kSetBytes);
            tma_load_3d(ring + slot * L::kSlotBytes, &tm, a_w - 1, b0 - 1 + k, c0 - 1, bar);
            if (IDT) tma_load_3d(ring + slot * L::kSlotBytes + L::kXBytes, &tm_ids, a_w - 3, b0 - 1 + k, c0 - id_plane0, bar);
        };
        auto prefetch = [&](int k) {  // the box of line set k into L2, PFD sets ahead of its fetch
            tma_prefetch_3d(&tm, a_w - 1, b0 - 1 + k, c0 - 1);
            if (IDT) tma_prefetch_3d(&tm_ids, a_w - 3, b0 - 1 + k, c0 - id_plane0);
        };
        if (lane == 0) {
            for (int k = 0; k < S && k < n_sets; k++) issue(k);
            if (PFD > 0 && PFD < 9)
                for (int k = S; k < S + PFD && k < n_sets; k++) prefetch(k);
        }
        if (!masks_staged) {
            for (int i = lane; i <= p.n_patterns; i += 32) sts_u32(s_masks + 4 * i, i == 0 ? 0u : p.masks[i - 1]);
            __syncwarp();
            masks_staged = true;
        }

        // per-thread geometry: columns a, a+1 (a odd); the row of (column a, line b0 + j, plane c0 + q) is row0 + q*sz + j*sy
        const int a = a_w + 2 * lane;
        const int64_t xi0 = a + (int64_t)sy * b0 + (int64_t)sz * c0;
        const int row0 = (int)(xi0 - p.g0);
        bool ok[Q][2];           // the row's column and plane exist
        uint32_t expect[Q][2];   // dictionary mask the plain chain is exact for, before the line term; 0 for rows that do not exist
#pragma unroll
        for (int q = 0; q < Q; q++) {
            const int c = c0 + q;
            const uint32_t oob_c = (c == 0 ? kDzLoBits : 0u) | (c == np_x - 1 ? kDzHiBits : 0u);
#pragma unroll
            for (int i = 0; i < 2; i++) {
                const uint32_t oob_a = (a + i == 0 ? kLBits : 0u) | (a + i == sy - 1 ? kRBits : 0u);
                ok[q][i] = a + i >= 0 && a + i < sy && c <= c_hi;
                expect[q][i] = (c >= np_x || !ok[q][i]) ? 0u : (kFullBox & ~(oob_a | oob_c));
            }
        }
        // The left-over column sy-1 (64 | sy) rides with the last strip: its operands -- columns sy-2, sy-1 of the three lines,
        // box elements 64 and 65; column sy is outside the view -- are in this warp's ring already, and so is its id (element
        // 67 of the id box).  Lane q < Q sums the row of plane c0+q after the strip's own rows, one short chain per step.
        const bool do_left = IDT && DBG == 0 && left_in_ring == 1 && strip == n_strips - 1;
        const int ql = min(lane, Q - 1);
        const int rowl0 = (int)((int64_t)(sy - 1) + (int64_t)sy * b0 + (int64_t)sz * (c0 + ql) - p.g0);
        const bool okl = do_left && lane < Q && c0 + ql <= c_hi;
        const uint32_t expect_l = (!okl || c0 + ql >= np_x) ? 0u
                                  : (kFullBox & ~(kRBits | (c0 + ql == 0 ? kDzLoBits : 0u) | (c0 + ql == np_x - 1 ? kDzHiBits : 0u)));
        // -1: no such row here (computed on whatever the ring holds, never stored)
        auto load_id = [&](int q, int i, int j) {
            const int r = row0 + q * sz + j * sy + i;
            return (ok[q][i] && j < nb && (unsigned)(r - rb) < n_range) ? __ldg(ids + r) : -1;
        };
        int idn[Q][2], idn2[Q][2];  // !IDT: the id stream is fetched two steps ahead into registers
        if (!IDT) {
#pragma unroll
            for (int q = 0; q < Q; q++)
#pragma unroll
                for (int i = 0; i < 2; i++) idn[q][i] = load_id(q, i, 0), idn2[q][i] = load_id(q, i, 1);
        }
        auto wait_set = [&](int k) { mbar_wait(bars + 8 * ((gs + k) % S), ((gs + k) / S) & 1); };
        wait_set(0);
        wait_set(1);
        if constexpr (LPS == 2) {
        // Two lines per step: the rows of lines b and b+1 (2 x Q x 2 per thread) from the line sets b-1 .. b+2 -- every operand quad
        // taken from shared memory serves both lines, 8 x P loads for 4Q rows instead of 6 x P for 2Q (the shared-memory data path
        // is this kernel's busiest unit).  A row still meets its entries in ascending (plane, line, column) order.  An odd march
        // ends with a step whose second line does not exist: computed on whatever the ring holds, never stored.
#pragma unroll 1
        for (int j = 0; j < nb; j += 2) {
            const int b = b0 + j;
            const bool two = j + 1 < nb;  // warp-uniform
            wait_set(j + 2);
            if (two) wait_set(j + 3);
            const bool lcopy = cta_left && strip == n_strips - 1;
            if (lcopy && j == 0) {
#pragma unroll 1
                for (int k = 0; k < 2; k++) {
                    const uint32_t src = ring + ((gs + k) % S) * L::kSlotBytes;
                    sts_f64x2(s_left + (k * P + min(lane, P - 1)) * 16, lds_f64x2(src + min(lane, P - 1) * L::kLineBytes + 64 * 8));
                    if (k == 1) sts_u32(s_left + L::kLeftXBytes + min(lane, Q - 1) * 4, lds_u32(src + L::kXBytes + min(lane, Q - 1) * L::kIdLineBytes + 67 * 4));
                }
            }
            uint32_t sl[4];
#pragma unroll
            for (int dy = 0; dy < 4; dy++) sl[dy] = ring + ((gs + j + dy) % S) * L::kSlotBytes + lane_off;
            int id[2][Q][2];
            uint32_t bad = 0;
            uint32_t in_b[2];
#pragma unroll
            for (int ln = 0; ln < 2; ln++) {
                in_b[ln] = ~((b + ln == 0 ? kDyLoBits : 0u) | (b + ln == pl - 1 ? kDyHiBits : 0u));
#pragma unroll
                for (int q = 0; q < Q; q++)
#pragma unroll
                    for (int i = 0; i < 2; i++) {
                        const int r = row0 + q * sz + (j + ln) * sy + i;
                        const int v = (int)lds_u32(sl[1 + ln] - lane_off + L::kXBytes + q * L::kIdLineBytes + (3 + 2 * lane + i) * 4);
                        id[ln][q][i] = (ok[q][i] && (ln == 0 || two) && (unsigned)(r - rb) < n_range) ? v : -1;
                        bad |= lds_u32(s_masks + 4 + 4 * id[ln][q][i]) ^ (expect[q][i] & in_b[ln]);  // id -1 reads entry 0 = 0
                    }
            }
            double acc[2][Q][2], xc[2][Q][2];
            {
#pragma unroll
                for (int ln = 0; ln < 2; ln++)
#pragma unroll
                    for (int q = 0; q < Q; q++) acc[ln][q][0] = acc[ln][q][1] = 0.0, xc[ln][q][0] = xc[ln][q][1] = 0.0;
                if (cpos == 0) {
#pragma unroll
                    for (int ln = 0; ln < 2; ln++)
#pragma unroll
                        for (int q = 0; q < Q; q++) {
                            const double2 u = lds_f64x2(sl[1 + ln] + (q + 1) * L::kLineBytes), v = lds_f64x2(sl[1 + ln] + (q + 1) * L::kLineBytes + 16);
                            acc[ln][q][0] = __dadd_rn(acc[ln][q][0], __dmul_rn(vc, u.y));
                            acc[ln][q][1] = __dadd_rn(acc[ln][q][1], __dmul_rn(vc, v.x));
                        }
                }
                double e[2][4][4];  // [buffer][line b-1 .. b+2][columns a-1 .. a+2]
                auto load_plane = [&](int buf, int pz) {
#pragma unroll
                    for (int ll = 0; ll < 4; ll++) {
                        const double2 u = lds_f64x2(sl[ll] + pz * L::kLineBytes), v = lds_f64x2(sl[ll] + pz * L::kLineBytes + 16);
                        e[buf][ll][0] = u.x, e[buf][ll][1] = u.y, e[buf][ll][2] = v.x, e[buf][ll][3] = v.y;
                    }
                };
                load_plane(0, 0);
#pragma unroll
                for (int pz = 0; pz < P; pz++) {
                    if (pz + 1 < P) load_plane((pz + 1) & 1, pz + 1);
#pragma unroll
                    for (int ll = 0; ll < 4; ll++)
#pragma unroll
                        for (int ln = 0; ln < 2; ln++) {
                            const int dy = ll - ln;
                            if (dy < 0 || dy > 2) continue;
#pragma unroll
                            for (int dx = 0; dx < 3; dx++)
#pragma unroll
                                for (int q = 0; q < Q; q++) {
                                    const int dz = pz - q;
                                    if (dz < 0 || dz > 2) continue;
                                    const int t = dz * 9 + dy * 3 + dx;
#pragma unroll
                                    for (int i = 0; i < 2; i++) {
                                        const double ev = e[pz & 1][ll][i + dx];
                                        if (t == 13) {
                                            xc[ln][q][i] = ev;
                                            if (cpos == 2) acc[ln][q][i] = __dadd_rn(acc[ln][q][i], __dmul_rn(vc, ev));
                                        } else if (OFF_NEG1) {
                                            acc[ln][q][i] = __dsub_rn(acc[ln][q][i], ev);
                                        } else {
                                            acc[ln][q][i] = __dadd_rn(acc[ln][q][i], __dmul_rn(vo, ev));
                                        }
                                    }
                                }
                        }
                }
                if (cpos == 1) {
#pragma unroll
                    for (int ln = 0; ln < 2; ln++)
#pragma unroll
                        for (int q = 0; q < Q; q++)
#pragma unroll
                            for (int i = 0; i < 2; i++) acc[ln][q][i] = __dadd_rn(acc[ln][q][i], __dmul_rn(vc, xc[ln][q][i]));
                }
            }
            if (__any_sync(0xffffffffu, bad != 0)) {  // see the one-line step below: masked sub-boxes, then List 1
#pragma unroll 1
                for (int ln = 0; ln < (two ? 2 : 1); ln++) {
                    uint32_t mk[Q * 2];
                    int idl_[Q * 2];
                    bool real = false;
#pragma unroll
                    for (int q = 0; q < Q; q++)
#pragma unroll
                        for (int i = 0; i < 2; i++) {
                            idl_[q * 2 + i] = ln == 0 ? id[0][q][i] : id[1][q][i];
                            mk[q * 2 + i] = lds_u32(s_masks + 4 + 4 * idl_[q * 2 + i]);
                            real = real || (idl_[q * 2 + i] >= 0 && mk[q * 2 + i] != (expect[q][i] & in_b[ln]));
                        }
                    if (__any_sync(0xffffffffu, real)) {
                        double am[Q * 2];
                        ring_masked_step<Q, OFF_NEG1, CENTER_POS, L::kLineBytes>(ln == 0 ? sl[0] : sl[1], ln == 0 ? sl[1] : sl[2], ln == 0 ? sl[2] : sl[3], mk, vc, vo, am,
                                                                                  p.center_pos);
#pragma unroll
                        for (int q = 0; q < Q; q++)
#pragma unroll
                            for (int i = 0; i < 2; i++) {
                                const uint32_t m = mk[q * 2 + i];
                                if (idl_[q * 2 + i] >= 0 && (m == kGenericMask || (m & ~(expect[q][i] & in_b[ln])) != 0))
                                    am[q * 2 + i] = pattern_row_cold(p, idl_[q * 2 + i], xi0 + (int64_t)(j + ln) * sy + (int64_t)q * sz + i);
                                if (ln == 0) acc[0][q][i] = am[q * 2 + i];
                                else acc[1][q][i] = am[q * 2 + i];
                            }
                    }
                }
            }
            double2 lx[2];
            uint32_t lid[2];
            if (lcopy) {  // what the left-over column needs of the two new line sets, before their predecessors' slots are refilled
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    const uint32_t src = ring + ((gs + j + 2 + k) % S) * L::kSlotBytes;
                    lx[k] = lds_f64x2(src + min(lane, P - 1) * L::kLineBytes + 64 * 8);
                    lid[k] = lds_u32(src + L::kXBytes + min(lane, Q - 1) * L::kIdLineBytes + 67 * 4);
                }
            }
            __syncwarp();  // every lane is done with the slots of lines b-1 and b
            if (lane == 0) {
                fence_proxy_async();  // generic-proxy reads before the async-proxy refill
                if (j + S < n_sets) issue(j + S);
                if (j + S + 1 < n_sets) issue(j + S + 1);
            }
#pragma unroll
            for (int ln = 0; ln < 2; ln++)
#pragma unroll
                for (int q = 0; q < Q; q++)
#pragma unroll
                    for (int i = 0; i < 2; i++)
                        if (id[ln][q][i] >= 0) {
                            y[row0 + q * sz + (j + ln) * sy + i] = acc[ln][q][i];
                            if (DOT) dsum = __dadd_rn(dsum, __dmul_rn(acc[ln][q][i], xc[ln][q][i]));  // the centre operand is the row's own x entry
                        }
            if (lcopy) {
                sts_f64x2(s_left + ((j + 2) * P + min(lane, P - 1)) * 16, lx[0]);
                if (j + 1 < nb) sts_u32(s_left + L::kLeftXBytes + ((j + 1) * Q + min(lane, Q - 1)) * 4, lid[0]);
                if (two) {
                    sts_f64x2(s_left + ((j + 3) * P + min(lane, P - 1)) * 16, lx[1]);
                    if (j + 2 < nb) sts_u32(s_left + L::kLeftXBytes + ((j + 2) * Q + min(lane, Q - 1)) * 4, lid[1]);
                }
            }
        }
        } else {
#pragma unroll 1
        for (int j = 0; j < nb; j++) {
            const int b = b0 + j;
            wait_set(j + 2);
            // The last strip's warp keeps what the left-over column needs of each line set in the CTA's side buffer -- columns sy-2,
            // sy-1 (box elements 64, 65) of every plane and the ids of column sy-1 (element 67 of the id box): loaded here, stored
            // behind the id / mask look-ups below so that no latency is exposed; the rows are summed by the whole CTA after the march.
            // (Fetching them from global memory instead -- 2 KB apart -- costs 3 us at 256^3, up front or spread over the steps alike.)
            const bool lcopy = cta_left && strip == n_strips - 1;
            double2 lx = make_double2(0.0, 0.0);
            uint32_t lid = 0;
            if (lcopy) {
                if (j == 0) {
#pragma unroll 1
                    for (int k = 0; k < 2; k++) {
                        const uint32_t src = ring + ((gs + k) % S) * L::kSlotBytes;
                        sts_f64x2(s_left + (k * P + min(lane, P - 1)) * 16, lds_f64x2(src + min(lane, P - 1) * L::kLineBytes + 64 * 8));
                        if (k == 1) sts_u32(s_left + L::kLeftXBytes + min(lane, Q - 1) * 4, lds_u32(src + L::kXBytes + min(lane, Q - 1) * L::kIdLineBytes + 67 * 4));
                    }
                }
            }
            uint32_t sl[3];
#pragma unroll
            for (int dy = 0; dy < 3; dy++) sl[dy] = ring + ((gs + j + dy) % S) * L::kSlotBytes + lane_off;
            if (DBG >= 3 && DBG <= 5) {  // measurement only: the data movement alone (ring fetches, waits, y stores)
                if (DBG == 3) {
                    const double2 u = lds_f64x2(sl[1] + L::kLineBytes);
#pragma unroll
                    for (int q = 0; q < Q; q++)
#pragma unroll
                        for (int i = 0; i < 2; i++)
                            if (ok[q][i]) y[row0 + q * sz + j * sy + i] = u.y;
                }
                __syncwarp();
                if (lane == 0 && j + S < n_sets) {
                    fence_proxy_async();
                    issue(j + S);
                }
                continue;
            }
            int id[Q][2];
            uint32_t bad = 0;
            const uint32_t in_b = ~((b == 0 ? kDyLoBits : 0u) | (b == pl - 1 ? kDyHiBits : 0u));
#pragma unroll
            for (int q = 0; q < Q; q++)
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    if (IDT) {  // set j+1 carries the ids of its line
                        const int r = row0 + q * sz + j * sy + i;
                        const int v = (int)lds_u32(sl[1] - lane_off + L::kXBytes + q * L::kIdLineBytes + (3 + 2 * lane + i) * 4);
                        id[q][i] = (ok[q][i] && (unsigned)(r - rb) < n_range) ? v : -1;
                    } else {
                        id[q][i] = idn[q][i];
                        idn[q][i] = idn2[q][i], idn2[q][i] = load_id(q, i, j + 2);
                    }
                    bad |= lds_u32(s_masks + 4 + 4 * id[q][i]) ^ (expect[q][i] & in_b);  // id -1 reads entry 0 = 0
                }
            double acc[Q][2];
            // The sums of the step.  Planes outermost, so that the Q rows of a thread consume each (plane, line) operand
            // quad together; the quads of plane pz+1 are fetched from shared memory while plane pz is being summed.
            {
                double xc[Q][2];
#pragma unroll
                for (int q = 0; q < Q; q++) acc[q][0] = acc[q][1] = 0.0;
                if (cpos == 0) {
#pragma unroll
                    for (int q = 0; q < Q; q++) {
                        const double2 u = lds_f64x2(sl[1] + (q + 1) * L::kLineBytes), v = lds_f64x2(sl[1] + (q + 1) * L::kLineBytes + 16);
                        acc[q][0] = __dadd_rn(acc[q][0], __dmul_rn(vc, u.y));
                        acc[q][1] = __dadd_rn(acc[q][1], __dmul_rn(vc, v.x));
                    }
                }
                double e[2][3][4];  // [buffer][dy][columns a-1 .. a+2]
                auto load_plane = [&](int buf, int pz) {
#pragma unroll
                    for (int dy = 0; dy < 3; dy++) {
                        if (DBG == 2 && !(pz == 1 && dy == 1)) {  // measurement only: one operand quad per step
                            e[buf][dy][0] = e[buf][dy][1] = e[buf][dy][2] = e[buf][dy][3] = vc;
                            continue;
                        }
                        const double2 u = lds_f64x2(sl[dy] + pz * L::kLineBytes), v = lds_f64x2(sl[dy] + pz * L::kLineBytes + 16);
                        e[buf][dy][0] = u.x, e[buf][dy][1] = u.y, e[buf][dy][2] = v.x, e[buf][dy][3] = v.y;
                    }
                };
                load_plane(0, 0);
#pragma unroll
                for (int pz = 0; pz < P; pz++) {
                    if (pz + 1 < P) load_plane((pz + 1) & 1, pz + 1);
#pragma unroll
                    for (int dy = 0; dy < 3; dy++)
#pragma unroll
                        for (int dx = 0; dx < 3; dx++)
#pragma unroll
                            for (int q = 0; q < Q; q++) {
                                const int dz = pz - q;
                                if (dz < 0 || dz > 2) continue;
                                const int t = dz * 9 + dy * 3 + dx;
#pragma unroll
                                for (int i = 0; i < 2; i++) {
                                    const double ev = e[pz & 1][dy][i + dx];
                                    if (t == 13) {
                                        if (cpos == 2) acc[q][i] = __dadd_rn(acc[q][i], __dmul_rn(vc, ev));
                                        else xc[q][i] = ev;
                                    } else if (DBG == 1) {  // measurement only: no dependent FP64 chain
                                        if (dx == 1 && dy == 1) acc[q][i] = __dsub_rn(acc[q][i], ev);
                                    } else if (OFF_NEG1) {
                                        acc[q][i] = __dsub_rn(acc[q][i], ev);
                                    } else {
                                        acc[q][i] = __dadd_rn(acc[q][i], __dmul_rn(vo, ev));
                                    }
                                }
                            }
                }
                if (cpos == 1) {
#pragma unroll
                    for (int q = 0; q < Q; q++)
#pragma unroll
                        for (int i = 0; i < 2; i++) acc[q][i] = __dadd_rn(acc[q][i], __dmul_rn(vc, xc[q][i]));
                }
            }
            if (__any_sync(0xffffffffu, bad != 0)) {
                // Some row the plain chain may not be exact for.  Sub-boxes whose entries are all inside the view (e.g. the
                // grid faces when x carries ghost planes beyond them): the sums again with every operand selected by the
                // row's mask.  Rows of other patterns, or with entries outside the view: List 1 as written.
                uint32_t mk[Q * 2];
                bool real = false;  // rows without an id (exception rows, range ends) raise the flag too, but need nothing
#pragma unroll
                for (int q = 0; q < Q; q++)
#pragma unroll
                    for (int i = 0; i < 2; i++) {
                        mk[q * 2 + i] = lds_u32(s_masks + 4 + 4 * id[q][i]);
                        real = real || (id[q][i] >= 0 && mk[q * 2 + i] != (expect[q][i] & in_b));
                    }
                if (__any_sync(0xffffffffu, real)) {
                    double am[Q * 2];
                    ring_masked_step<Q, OFF_NEG1, CENTER_POS, L::kLineBytes>(sl[0], sl[1], sl[2], mk, vc, vo, am, p.center_pos);
#pragma unroll
                    for (int q = 0; q < Q; q++)
#pragma unroll
                        for (int i = 0; i < 2; i++) {
                            const uint32_t m = mk[q * 2 + i];
                            if (id[q][i] >= 0 && (m == kGenericMask || (m & ~(expect[q][i] & in_b)) != 0))
                                am[q * 2 + i] = pattern_row_cold(p, id[q][i], xi0 + (int64_t)j * sy + (int64_t)q * sz + i);
                            acc[q][i] = am[q * 2 + i];
                        }
                }
            }
            double accl = 0.0, xcl = 0.0;
            int idl = -1;
            if (do_left) {  // warp-uniform
                const int rl = rowl0 + j * sy;
                const int v = (int)lds_u32(sl[1] - lane_off + L::kXBytes + ql * L::kIdLineBytes + 67 * 4);
                idl = (okl && (unsigned)(rl - rb) < n_range) ? v : -1;
                const uint32_t lb = sl[0] - lane_off + ql * L::kLineBytes + 64 * 8, lc = sl[1] - lane_off + ql * L::kLineBytes + 64 * 8,
                               lt = sl[2] - lane_off + ql * L::kLineBytes + 64 * 8;
                xcl = lds_f64(lc + L::kLineBytes + 8);
                if (cpos == 0) accl = __dadd_rn(accl, __dmul_rn(vc, xcl));
#pragma unroll
                for (int dz = 0; dz < 3; dz++)
#pragma unroll
                    for (int dy = 0; dy < 3; dy++) {
                        const double2 u = lds_f64x2((dy == 0 ? lb : dy == 1 ? lc : lt) + dz * L::kLineBytes);
                        accl = OFF_NEG1 ? __dsub_rn(accl, u.x) : __dadd_rn(accl, __dmul_rn(vo, u.x));
                        if (dz == 1 && dy == 1) {
                            if (cpos == 2) accl = __dadd_rn(accl, __dmul_rn(vc, u.y));
                        } else {
                            accl = OFF_NEG1 ? __dsub_rn(accl, u.y) : __dadd_rn(accl, __dmul_rn(vo, u.y));
                        }
                    }
                if (cpos == 1) accl = __dadd_rn(accl, __dmul_rn(vc, xcl));
                // any other row shape (or entries outside the view): List 1 as written
                if (idl >= 0 && lds_u32(s_masks + 4 + 4 * idl) != (expect_l & in_b))
                    accl = pattern_row_cold(p, idl, (int64_t)rl + p.g0);
            }
            __syncwarp();  // every lane is done with the slot of line b-1
            if (lane == 0 && j + S < n_sets) {
                fence_proxy_async();  // generic-proxy reads before the async-proxy refill
                issue(j + S);
                if (PFD > 0 && PFD < 9 && j + S + PFD < n_sets) prefetch(j + S + PFD);
            }
            if (idl >= 0) {
                y[rowl0 + j * sy] = accl;
                if (DOT) dsum = __dadd_rn(dsum, __dmul_rn(accl, xcl));
            }
            if (lcopy) {  // loaded here, stored behind the y stores below: the shared-memory stores then sit at the end of the step, next
                          // to the fences of the refill, and leave the scheduling of the step's loads alone
                const uint32_t src = ring + ((gs + j + 2) % S) * L::kSlotBytes;
                lx = lds_f64x2(src + min(lane, P - 1) * L::kLineBytes + 64 * 8);
                lid = lds_u32(src + L::kXBytes + min(lane, Q - 1) * L::kIdLineBytes + 67 * 4);
            }
            // (16-byte stores of the aligned pairs (a+1, a+2) through a lane shuffle were measured slower: 81 vs 78 us)
#pragma unroll
            for (int q = 0; q < Q; q++)
#pragma unroll
                for (int i = 0; i < 2; i++)
                    if (id[q][i] >= 0) {
                        if (PFD == 9) __stcs(&y[row0 + q * sz + j * sy + i], acc[q][i]);
                        else y[row0 + q * sz + j * sy + i] = acc[q][i];
                        // the row's own x entry is still in the ring (line b, plane q of the box + 1; the refill above took line b-1)
                        if (DOT) dsum = __dadd_rn(dsum, __dmul_rn(acc[q][i], lds_f64(sl[1] + (q + 1) * L::kLineBytes + 8 * (1 + i))));
                    }
            if (lcopy) {
                sts_f64x2(s_left + ((j + 2) * P + min(lane, P - 1)) * 16, lx);
                if (j + 1 < nb) sts_u32(s_left + L::kLeftXBytes + ((j + 1) * Q + min(lane, Q - 1)) * 4, lid);
            }
        }
        }  // LPS
        gs += n_sets;
        __syncwarp();
        }
        if (cta_left) {
            // The rows of column sy-1 of this march, dealt out to all threads: same sums, same exactness rule as the strips' rows.
            if (!masks_staged) {
                for (int i = lane; i <= p.n_patterns; i += 32) sts_u32(s_masks + 4 * i, i == 0 ? 0u : p.masks[i - 1]);
                masks_staged = true;
            }
            __syncthreads();
            for (int t = threadIdx.x; t < nb * Q; t += kRingWarps * 32) {
                const int idl = (int)lds_u32(s_left + L::kLeftXBytes + t * 4);
                const int ll = t / Q, q = t - ll * Q;
                const int line = b0 + ll, c = c0 + q;
                const int rl = (int)((int64_t)(sy - 1) + (int64_t)sy * line + (int64_t)sz * c - p.g0);
                if (idl < 0 || c > c_hi || (unsigned)(rl - rb) >= n_range) continue;
                const uint32_t base = s_left + (ll * P + q) * 16;  // (line b0+ll-1, plane c-1): the row's entry dy = dz = -1
                const double xcl = lds_f64x2(base + (P + 1) * 16).y;
                double accl = 0.0;
                if (cpos == 0) accl = __dadd_rn(accl, __dmul_rn(vc, xcl));
#pragma unroll
                for (int dz = 0; dz < 3; dz++)
#pragma unroll
                    for (int dy = 0; dy < 3; dy++) {
                        const double2 u = lds_f64x2(base + (dy * P + dz) * 16);
                        accl = OFF_NEG1 ? __dsub_rn(accl, u.x) : __dadd_rn(accl, __dmul_rn(vo, u.x));
                        if (dz == 1 && dy == 1) {
                            if (cpos == 2) accl = __dadd_rn(accl, __dmul_rn(vc, u.y));
                        } else {
                            accl = OFF_NEG1 ? __dsub_rn(accl, u.y) : __dadd_rn(accl, __dmul_rn(vo, u.y));
                        }
                    }
                if (cpos == 1) accl = __dadd_rn(accl, __dmul_rn(vc, xcl));
                const uint32_t exp_l = c >= np_x ? 0u
                                                 : (kFullBox & ~(kRBits | (c == 0 ? kDzLoBits : 0u) | (c == np_x - 1 ? kDzHiBits : 0u) |
                                                                 (line == 0 ? kDyLoBits : 0u) | (line == pl - 1 ? kDyHiBits : 0u)));
                // any other row shape (or entries outside the view): List 1 as written
                if (lds_u32(s_masks + 4 + 4 * idl) != exp_l) accl = pattern_row_cold(p, idl, (int64_t)rl + p.g0);
                y[rl] = accl;
                if (DOT) dsum = __dadd_rn(dsum, __dmul_rn(accl, xcl));
            }
            __syncthreads();  // the buffer is free for the next march
        }
    }
    {  // this warp's share of the left-over columns (after its marches: the warps do not finish in step, so these
       // latency-bound gathers overlap with the marches of the others)
        const int n_left = sy - left_lo;
        const int total_left = n_left * pl * (c_hi - c_lo + 1);
        if (!masks_staged && n_left > 0) {  // a warp without a march
            for (int i = lane; i <= p.n_patterns; i += 32) sts_u32(s_masks + 4 * i, i == 0 ? 0u : p.masks[i - 1]);
            __syncwarp();
        }
        for (int t = gw * 32 + lane; t < total_left && DBG != 5 && DBG != 6; t += n_warps * 32) {
            const double d = ring_leftover_row<OFF_NEG1, CENTER_POS>(p, s_masks, left_lo + t % n_left, (t / n_left) % pl, c_lo + t / (n_left * pl), np_x);
            if (DOT) dsum = __dadd_rn(dsum, d);
        }
    }
    if (DOT) {  // one partial per warp, fixed tree
        for (int o = 16; o > 0; o >>= 1) dsum = __dadd_rn(dsum, __shfl_down_sync(0xffffffffu, dsum, o));
        if (lane == 0) p.dot_partial[gw] = dsum;
    }
}

// ---- host side ------------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                                   const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            ptr = nullptr;
        return reinterpret_cast<EncodeTiledFn>(ptr);
    }();
    return fn;
}

// A [planes][plane_lines lines][sy columns] view of `base` with a box of box_cols x 1 x box_planes elements
// (x: fp64, 68 columns, Q+2 planes; ids: int32, 72 columns, Q planes).  One cached map per thread and kind.
static int make_view_map(int kind, const void *base, int sy, int pl, int planes, int box_cols, int box_planes, CUtensorMap *out) {
    struct Key {
        const void *base;
        int sy, pl, np, bc, bp;
    };
    thread_local Key last[2] = {{nullptr, 0, 0, 0, 0, 0}, {nullptr, 0, 0, 0, 0, 0}};
    thread_local CUtensorMap last_map[2];
    Key &k = last[kind];
    if (k.base == base && k.sy == sy && k.pl == pl && k.np == planes && k.bc == box_cols && k.bp == box_planes) {
        *out = last_map[kind];
        return SPMVB_OK;
    }
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return fail(SPMVB_ERR_CUDA, "cuTensorMapEncodeTiled is not available from this driver");
    const cuuint64_t esz = kind == 0 ? 8 : 4;
    const cuuint64_t dims[3] = {(cuuint64_t)sy, (cuuint64_t)pl, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)sy * esz, (cuuint64_t)sy * pl * esz};
    const cuuint32_t box[3] = {(cuuint32_t)box_cols, 1u, (cuuint32_t)box_planes};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(&last_map[kind], kind == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_INT32, 3,
                           const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        k.base = nullptr;
        return fail(SPMVB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) for view %d x %d x %d", (int)r, planes, pl, sy);
    }
    k = Key{base, sy, pl, planes, box_cols, box_planes};
    *out = last_map[kind];
    return SPMVB_OK;
}

// The view of x only needs the planes that hold columns the matrix references.  Planes before / after them (e.g. the
// ghost planes a slab layout keeps beyond the faces of the global grid) are cut off, so that the entries the face
// rows lack fall outside the view -- zero-filled, i.e. the plain chain is exact there too.  Shifts x / g0 / x_len of
// a copy of the arguments by whole planes; every consumer (List 1 included) stays consistent.
static PatternArgs clip_view(const spmvb_matrix *a, const PatternArgs &p) {
    PatternArgs q = p;
    if (a->col_max < a->col_min) return q;
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    const int64_t x_col0 = a->row_offset - p.g0;
    const int64_t lo = std::max<int64_t>(0, a->col_min - x_col0), hi = std::min<int64_t>(p.x_len - 1, a->col_max - x_col0);
    if (hi < lo) return q;
    const int64_t k_lo = lo / sz;
    int64_t planes = hi / sz - k_lo + 1;
    if ((k_lo + planes) * sz > p.x_len) planes = (p.x_len - k_lo * sz) / sz;  // whole planes only
    if (planes < 1 || p.g0 - k_lo * sz + p.row_begin < 0) return q;
    q.x = p.x + k_lo * sz;
    q.g0 = p.g0 - k_lo * sz;
    q.x_len = planes * sz;
    return q;
}

// The id stream can ride through the ring when its rows form whole planes of the same view: g0 a multiple of the
// plane, a whole number of planes of rows, 16-byte aligned base and line stride.
static bool ids_view_ok(const spmvb_matrix *a, const PatternArgs &p) {
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    return p.g0 >= 0 && p.g0 % sz == 0 && (int64_t)a->n % sz == 0 && p.sy % 4 == 0 && (uintptr_t)p.ids % 16 == 0;
}

template <int Q, int S, int MINB, bool IDT, int PFD = 0, int DBG = 0, bool CTAC = false, bool DOT = false, int LPS = 1>
static int launch_ringp_t(const spmvb_matrix *a, PatternArgs &p_in, int chunk, cudaStream_t st, int tile_lines = 0) {
    PatternArgs p = clip_view(a, p_in);
    using L = RingLayout<Q, S, IDT, LPS>;
    const bool neg1 = p.v_off == -1.0;
    const int cp = a->box.center_pos;
    if (IDT && !ids_view_ok(a, p)) return 1;
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    const int np_x = (int)(p.x_len / sz);
    const int c_lo = (int)((p.g0 + p.row_begin) / sz), c_hi = (int)((p.g0 + p.row_end - 1) / sz);
    const int id_plane0 = (int)(p.g0 / sz);
    CUtensorMap tm, tm_ids;
    if (make_view_map(0, p.x, p.sy, p.plane_lines, np_x, kBoxCols, Q + 2, &tm) != SPMVB_OK) return -1;
    if (IDT) {
        if (make_view_map(1, p.ids, p.sy, p.plane_lines, (int)(a->n / sz), kIdBoxCols, Q, &tm_ids) != SPMVB_OK) return -1;
    } else {
        tm_ids = tm;  // unused
    }
    int n_strips = (p.sy + 1) / kStripCols;
    if (p.sy - (n_strips * kStripCols - 1) > 2) n_strips++;
    int left_lo = std::min(p.sy, n_strips * kStripCols - 1);
    // one left-over column (64 | sy) and ids through the ring: the last strip's warp sums it from its own ring
    int left_in_ring = (IDT && DBG == 0 && p.sy - left_lo == 1 && options().ring_leftover != 1) ? 1 : 0;
    if (left_in_ring) left_lo = p.sy;
    // ... or, in the chunk-per-CTA kernels, the whole CTA sums it at the end of each march (2; ring_leftover = 2 keeps the per-step sums)
    constexpr bool kFlush = RING_LEFT_MODE == 1 && IDT && DBG == 0 && CTAC;
    if (kFlush && left_in_ring && options().ring_leftover != 2 && tile_lines <= L::kLeftCap) left_in_ring = 2;
    if (LPS == 2 && left_in_ring == 1) return 1;  // the two-line step does not carry the per-step sums of the left-over column
    constexpr uint32_t kSmem = L::kTotal + (kFlush ? L::kLeftBytes : 0u);
    const int n_cols = CTAC ? (n_strips + kRingWarps - 1) / kRingWarps : n_strips;
    const int units = CTAC ? 1 : kRingWarps;  // chunks per CTA
    const int64_t total64 = (int64_t)n_cols * ((c_hi - c_lo + Q) / Q) * p.plane_lines;
    if (total64 >= INT32_MAX) return 1;
    const int total = (int)total64;
    static PerDevice<int> n_sm_dev;
    int &n_sm = n_sm_dev.get();
    if (n_sm == 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    }
    // one wave of CTAs; every warp gets the same number of line steps (at least `min_steps`, so that small problems
    // do not pay two halo line sets for a handful of steps)
    // (128^3: 14.8 us with 8, 13.5 us with 2-4: a full wave, launched with PDL.  Hybrid handles keep 8: their exception block
    // runs beside this kernel on a second stream and needs room on the SMs -- C4 at 128^3: 41.6 vs 49.8 us)
    const int min_steps = options().ring_min_steps > 0 ? options().ring_min_steps : (a->n_exc > 0 ? 8 : 4);
#define LAUNCH_RINGP(NEG, CP)                                                                                                   \
    do {                                                                                                                         \
        static PerDevice<int> per_sm_dev;                                                                                        \
        int &per_sm = per_sm_dev.get();                                                                                          \
        if (per_sm == 0) {                                                                                                       \
            if (cudaFuncSetAttribute(spmv_pattern_ringp_kernel<Q, S, MINB, NEG, CP, IDT, PFD, DBG, CTAC, DOT, LPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     (int)kSmem) != cudaSuccess ||                                                               \
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmv_pattern_ringp_kernel<Q, S, MINB, NEG, CP, IDT, PFD, DBG, CTAC, DOT, LPS>,      \
                                                              kRingWarps * 32, kSmem) != cudaSuccess || per_sm <= 0)             \
                return -1;                                                                                                       \
        }                                                                                                                        \
        int grid = n_sm * per_sm;                                                                                                \
        if (tile_lines > 0) {                                                                                                    \
            const int n_tiles = n_cols * ((c_hi - c_lo + Q) / Q) * ((p.plane_lines + tile_lines - 1) / tile_lines);              \
            grid = std::max(1, std::min(grid, (n_tiles + units - 1) / units));                                                   \
        } else                                                                                                                   \
            grid = std::max(1, std::min(grid, (total + min_steps * units - 1) / (min_steps * units)));                          \
        /* equal shares: total = (grid * units) * spw + rem, the first rem units take one step more (a forced chunk length:  */ \
        /* as many units as it needs)                                                                                       */ \
        int spw = chunk > 0 ? chunk : total / (grid * units), rem = chunk > 0 ? 0 : total - spw * (grid * units);                \
        if (spw == 0) spw = 1, rem = 0, grid = (total + units - 1) / units;                                                      \
        if (chunk > 0) grid = (total + spw * units - 1) / (spw * units);                                                         \
        const int cols_per_group = CTAC ? n_cols : n_strips;                                                                    \
        const int64_t wgrp = (int64_t)cols_per_group * p.plane_lines, kgrp = (wgrp + spw / 2) / spw;                              \
        const int rot = (kLabBuild && options().debug_nochain == 7) ? 0 : (int)(((wgrp - kgrp * spw) % p.plane_lines + p.plane_lines) % p.plane_lines); \
        if (DOT) {                                                                                                               \
            if (grid * kRingWarps > p.dot_capacity) return 1;                                                                    \
            fused_dot_request()->count = grid * kRingWarps;                                                                      \
        }                                                                                                                        \
        cudaLaunchConfig_t cfg = {};                                                                                             \
        cfg.gridDim = dim3(grid);                                                                                                \
        cfg.blockDim = dim3(kRingWarps * 32);                                                                                    \
        cfg.dynamicSmemBytes = kSmem;                                                                                            \
        cfg.stream = st;                                                                                                         \
        cudaLaunchAttribute pdl[1];                                                                                              \
        pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                                          \
        pdl[0].val.programmaticStreamSerializationAllowed = 1;                                                                   \
        cfg.attrs = pdl;                                                                                                         \
        cfg.numAttrs = (options().ring_pdl && grid == n_sm * per_sm) ? 1 : 0; /* only a full wave: early CTAs of a partial grid crowd the SMs that free up first (128^3: 14.2 -> 17.9 us) */                                                                               \
        if (cudaLaunchKernelEx(&cfg, spmv_pattern_ringp_kernel<Q, S, MINB, NEG, CP, IDT, PFD, DBG, CTAC, DOT, LPS>, tm, tm_ids, p, c_lo, c_hi, np_x,     \
                               n_strips, left_lo, left_in_ring, id_plane0, total, spw, rem, tile_lines, rot) != cudaSuccess)          \
            return check_launch("spmv_pattern_ringp") == SPMVB_OK ? -1 : -1;                                                     \
    } while (0)
    // two instantiations: the HPCG value pattern (off-diagonals -1, centre last) fully specialised, and a general one
    // (any off-diagonal value -- a product by -1.0 is exact, so it serves that case too -- centre position read at run time)
    if (neg1 && cp == 1) LAUNCH_RINGP(true, 1);
    else if constexpr (LPS == 2) return 1;  // the two-lines step is built for the stencil's value pattern only; the caller runs the one-line kernels
    else LAUNCH_RINGP(false, -1);
#undef LAUNCH_RINGP
    return check_launch("spmv_pattern_ringp") == SPMVB_OK ? 0 : -1;
}

#ifdef SPMVB_RING_TU_Q6
// Second translation unit (spmv_pattern_tma6.cu): the 6-planes-per-thread instantiations, so that the two halves build in parallel.
// mode 0: chunk per CTA (with the ids-by-loads fallback); 1: per CTA, lab; 2: per warp, lab; 3-5: ablations.
int launch_ring_q6(int mode, const spmvb_matrix *a, PatternArgs &p, int chunk, cudaStream_t st, int tile_lines) {
    if (mode == 6) return launch_ringp_t<4, 6, 2, true, 0, 0, true, false, 2>(a, p, chunk, st, tile_lines);  // 4 planes x 2 lines per thread and step, per CTA
    if (mode == 2) return launch_ringp_t<6, 4, 2, true>(a, p, chunk, st, tile_lines);  // a chunk per warp (strips that do not come in fours)
#ifdef SPMVB_LAB
    if (mode == 3) return launch_ringp_t<6, 4, 2, true, 0, 6, true>(a, p, chunk, st, tile_lines);  // measurement only: no left-over columns
    if (mode == 4) return launch_ringp_t<6, 4, 2, true, 0, 3, true>(a, p, chunk, st, tile_lines);  // measurement only: fetch + store
    if (mode == 5) return launch_ringp_t<6, 4, 2, true, 0, 4, true>(a, p, chunk, st, tile_lines);  // measurement only: fetch
#endif
    if (mode == 0 && p.dot_partial && fused_dot_request()) {  // cg_solve: x.y in the same pass (ids through the ring only)
        const int rcd = launch_ringp_t<6, 4, 2, true, 0, 0, true, true>(a, p, chunk, st, tile_lines);
        if (rcd != 1) return rcd;
        fused_dot_request()->count = 0;
    }
    const int rc = launch_ringp_t<6, 4, 2, true, 0, 0, true>(a, p, chunk, st, tile_lines);
    return rc == 1 && mode == 0 ? launch_ringp_t<6, 5, 2, false, 0, 0, true>(a, p, chunk, st, tile_lines) : rc;
}
// The 4-planes-per-thread kernels of the default policy with the fused dot (cg_solve); 1 = not served, run the plain kernel.
int launch_ring_q4_dot(bool per_cta, const spmvb_matrix *a, PatternArgs &p, int chunk, cudaStream_t st, int tile_lines) {
    if (!p.dot_partial || !fused_dot_request()) return 1;
    const int rc = per_cta ? launch_ringp_t<4, 4, 3, true, 0, 0, true, true>(a, p, chunk, st, tile_lines)
                           : launch_ringp_t<4, 4, 3, true, 0, 0, false, true>(a, p, chunk, st, tile_lines);
    if (rc == 1) fused_dot_request()->count = 0;
    return rc;
}
#else
int launch_ring_q6(int mode, const spmvb_matrix *a, PatternArgs &p, int chunk, cudaStream_t st, int tile_lines);
int launch_ring_q4_dot(bool per_cta, const spmvb_matrix *a, PatternArgs &p, int chunk, cudaStream_t st, int tile_lines);

// Conditions: the TMA view needs a 16-byte aligned base, strides that are multiples of 16 bytes (even
// sy), at least one whole plane of x and a line no narrower than a box; row arithmetic is 32-bit.
bool ring_ok(const spmvb_matrix *a, const PatternArgs &p) {
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    return (p.sy % 2 == 0) && p.sy >= kBoxCols && ((uintptr_t)p.x % 16 == 0) && a->n_patterns <= kDictSmemPat && p.x_len >= sz &&
           p.g0 + p.row_begin >= 0 && sz < (1 << 28) && p.x_len / sz < (1 << 30) && (int64_t)a->n + 2 * sz < INT32_MAX &&
           p.g0 > -(int64_t)INT32_MAX / 2 && p.g0 < INT32_MAX / 2;
}

// which: 0 = default configuration; others are measured alternatives and ablations (profiles/r01_probe256_ring_ablations.log,
// r01_probe_shapes_tensor_ring.log).  `lines` = chunk length (contiguous schedule) or tile length (round-robin schedule).
int launch_pattern_ring(int which, int lines, const spmvb_matrix *a, PatternArgs &p, cudaStream_t st) {
    int rc = 1;
    const int tl = lines > 0 ? lines : 16;
    switch (which) {
#ifdef SPMVB_LAB
        case 6: return launch_ringp_t<4, 4, 3, true, 2>(a, p, lines, st);     // + TMA L2 prefetch 2 sets ahead: 95 us (4 ahead: 105 us)
        case 7: return launch_ringp_t<4, 4, 3, true, 0, 1>(a, p, lines, st);  // measurement only (wrong results): no FP64 chains
        case 8: return launch_ringp_t<4, 4, 3, true, 0, 2>(a, p, lines, st);  // measurement only (wrong results): one operand quad per step
        case 9: return launch_ringp_t<4, 4, 3, true, 0, 3>(a, p, lines, st);  // measurement only: ring fetches + y stores, nothing else
        case 10: return launch_ringp_t<4, 4, 3, true, 0, 4>(a, p, lines, st); // measurement only: ring fetches only
        case 12: return launch_ringp_t<4, 4, 3, true, 0, 4, true>(a, p, lines, st);  // CTA chunks, fetch only
        case 13: return launch_ringp_t<4, 4, 3, true, 0, 3, true>(a, p, lines, st);  // CTA chunks, fetch + store only
        case 14:  // CTA chunks, 2 planes/thread, 6 slots: 90 us
            rc = launch_ringp_t<2, 6, 3, true, 0, 0, true>(a, p, lines, st);
            return rc == 1 ? launch_ringp_t<4, 5, 3, false, 0, 0, true>(a, p, lines, st) : rc;
        case 15: return launch_ringp_t<4, 4, 3, true, 9, 0, true>(a, p, lines, st);   // CTA chunks, streaming (evict-first) y stores: no change
        case 16: return launch_ringp_t<4, 4, 3, true, 0, 5, true>(a, p, lines, st);   // measurement only: fetch only, no left-over columns
        case 25: return launch_ring_q6(1, a, p, 0, st, tl);      // 6 planes/thread, round-robin tiles per CTA
        case 26: return launch_ring_q6(2, a, p, lines, st, 0);   // 6 planes/thread, chunk per warp
        case 28: return launch_ring_q6(3, a, p, lines, st, 0);   // ablations of the default (6 planes/thread, chunk per CTA):
        case 29: return launch_ring_q6(4, a, p, lines, st, 0);   //   no left-over columns / fetch + store only / fetch only
        case 30: return launch_ring_q6(5, a, p, lines, st, 0);
        case 27: return launch_ring_q6(2, a, p, 0, st, tl);      // 6 planes/thread, round-robin tiles per warp
#endif
        // the schedules the default policy chooses between, forced (tests cover each of them on every shape):
        case 21:  // two lines per step (4 planes/thread, 6 slots, 8 warps/SM), chunk per CTA: 70.6 us at 256^3
        case 22:  // ... tiles of `lines` lines dealt out round-robin (the default for x far beyond L2: 512^3 547-555 vs 577-581 us)
            rc = which == 21 ? launch_ring_q6(6, a, p, lines, st, 0) : launch_ring_q6(6, a, p, 0, st, lines > 0 ? lines : 28);
            if (rc != 1) return rc;
            rc = launch_ringp_t<4, 4, 3, true, 0, 0, true>(a, p, which == 21 ? lines : 0, st, which == 21 ? 0 : tl);
            return rc == 1 ? launch_ringp_t<4, 5, 3, false, 0, 0, true>(a, p, which == 21 ? lines : 0, st, which == 21 ? 0 : tl) : rc;
        case 11:  // a chunk per warp instead of per CTA: 87 us
            rc = launch_ringp_t<4, 4, 3, true>(a, p, lines, st);
            return rc == 1 ? launch_ringp_t<4, 5, 3, false>(a, p, lines, st) : rc;
        case 17: return launch_ringp_t<4, 5, 3, false, 0, 0, true>(a, p, lines, st);  // CTA chunks, 5 slots, ids by per-thread loads: 81 us
        case 18:  // tiles of `lines` (default 16) lines dealt out round-robin, a tile per CTA: 85-87 us (512^3: 530-575 us)
            rc = launch_ringp_t<4, 4, 3, true, 0, 0, true>(a, p, 0, st, tl);
            return rc == 1 ? launch_ringp_t<4, 5, 3, false, 0, 0, true>(a, p, 0, st, tl) : rc;
        case 20:  // 4 planes/thread, 12 warps/SM, chunk per CTA (the default before 6 planes/thread): 77 us
            rc = launch_ringp_t<4, 4, 3, true, 0, 0, true>(a, p, lines, st);
            return rc == 1 ? launch_ringp_t<4, 5, 3, false, 0, 0, true>(a, p, lines, st) : rc;
        // (3 / 5 / 7 / 8 planes per thread, chunk per CTA: 80.6 / 76.2 / 74.0 / 84.1 us at 256^3, r01_probe_planes_per_thread.log)
        // (small L2-resident grids, a chunk per warp: 2 planes/thread with 8 or 6 slots, 4 planes/thread with 6 slots -- 15.5 / 15.7 /
        //  14.8 us at 128^3 against 14.2 us for the default: measured and removed)
        case 19:  // ... a tile per warp
            rc = launch_ringp_t<4, 4, 3, true>(a, p, 0, st, tl);
            return rc == 1 ? launch_ringp_t<4, 5, 3, false>(a, p, 0, st, tl) : rc;
        default: {
            // One wave of persistent CTAs; ids through the ring when their rows are whole planes of the view, else two steps
            // ahead in registers.  Schedule and planes per thread (measured per shape,
            // profiles/r01_probe_shapes_tensor_ring.log, r01_probe_planes_per_thread.log):
            //  * x (about) fits L2: the (strip group, plane group) x line sequence cut into equal contiguous chunks -- per CTA
            //    with its warps on the four strips of the same lines when the strips come in fours (6 planes/thread, 8 warps/SM:
            //    73 us at 256^3; 4 planes/thread, 12 warps/SM: 77 us), else per warp with 4 planes/thread (and only while x is
            //    well inside L2);
            //  * larger x: tiles of 16 lines, columns fastest, dealt out round-robin, which keeps the planes being read few
            //    enough for their halo planes to be re-read from L2 (512^3: 530-575 us vs 686 us with contiguous chunks).
            static PerDevice<int> l2_dev;
            int &l2_bytes = l2_dev.get();
            if (l2_bytes == 0) {
                int dev = 0;
                if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&l2_bytes, cudaDevAttrL2CacheSize, dev) != cudaSuccess) return -1;
            }
            int n_strips = (p.sy + 1) / kStripCols;
            if (p.sy - (n_strips * kStripCols - 1) > 2) n_strips++;
            const bool fours = n_strips % kRingWarps == 0;
            const double x_bytes = (double)p.x_len * 8.0;
            const int tile_lines = (x_bytes > 1.25 * l2_bytes || (!fours && x_bytes > 0.8 * l2_bytes)) ? tl : 0;
            const int chunk = tile_lines ? 0 : lines;
            if (fours && tile_lines == 0) {  // 6 planes/thread at 8 warps/SM: 5-10 % faster than 4 at 12 on every shape tried
                return launch_ring_q6(0, a, p, chunk, st, 0);
            }
            rc = launch_ring_q4_dot(fours, a, p, chunk, st, tile_lines);  // cg_solve's request for x.y, when there is one
            if (rc != 1) return rc;
            // x far beyond L2 and strips in fours: two lines per step, tiles of 28 lines (what the side buffer of the left-over column
            // holds).  There the kernel's own shared-memory traffic, not the halo planes' L2 traffic, is the larger term: a quad of
            // operands serves the rows of two lines (23 instead of 29 L1 wavefronts per row).  512^3: 547-555 us against 577-581 us in
            // the same run; with x in L2 (256^3: 70.6 vs 65.9 us for 6 planes per thread) or strips not in fours (384^3) it loses.
            if (fours && tile_lines > 0 && a->n_exc == 0 && options().ring_two_lines) {
                rc = launch_ring_q6(6, a, p, 0, st, lines > 0 ? lines : 28);
                if (rc != 1) return rc;
            }
            // 6 planes/thread with a chunk per warp (128^3 13.5 -> 12.8 us, 192^3 33.9 -> 32.4 us) when every warp of its full wave
            // gets at least 4 steps (96^3 does not: 8.6 -> 10.4 us) and no exception block wants room beside it (C4: 41.9 -> 43.3 us)
            if (!fours && tile_lines == 0 && a->n_exc == 0) {
                static PerDevice<int> sm_dev;
                int &sms = sm_dev.get();
                if (sms == 0) {
                    int dev = 0;
                    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
                }
                const int64_t sz = (int64_t)p.sy * p.plane_lines;
                const int64_t planes = ((int64_t)p.row_end - p.row_begin + sz - 1) / sz;
                const int64_t steps6 = (int64_t)n_strips * ((planes + 5) / 6) * p.plane_lines;
                if (steps6 >= 4LL * 2 * sms * kRingWarps) {
                    rc = launch_ring_q6(2, a, p, chunk, st, 0);
                    if (rc != 1) return rc;
                }
            }
            if (fours) {
                rc = launch_ringp_t<4, 4, 3, true, 0, 0, true>(a, p, chunk, st, tile_lines);
                return rc == 1 ? launch_ringp_t<4, 5, 3, false, 0, 0, true>(a, p, chunk, st, tile_lines) : rc;
            }
            rc = launch_ringp_t<4, 4, 3, true>(a, p, chunk, st, tile_lines);
            return rc == 1 ? launch_ringp_t<4, 5, 3, false>(a, p, chunk, st, tile_lines) : rc;
        }
    }
}

#endif  // SPMVB_RING_TU_Q6

}  // namespace spmvb
