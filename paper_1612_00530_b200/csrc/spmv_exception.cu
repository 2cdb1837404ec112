// Exception rows of the hybrid pattern format (the paper's partial compression):
// rows without a dictionary pattern are kept uncompressed in an ELL block (n_exc x w_exc, slot order = ascending column,
// SPEC.md:208-211) and summed in slot order, y[exc_rows[e]] = sum_k v[e,k] * x[c[e,k]] -- bit-identical to the ELL kernel.
//
// Why not the ELL kernel with a row map (round 1: 41 us for the 209,894 exception rows of BASELINE config 4, 2.3 TB/s):
// exception rows are scattered over the grid (one row in ten), so every gather instruction of a thread-per-row tile touches
// ~28 different 32-byte sectors of x, 15 of them L1 misses per row; ncu shows the kernel waiting on those sector requests
// (issue slots 10 % busy, DRAM 29 %).  But the rows of a tile are *near* each other: 64 consecutive exception rows span
// ~640 grid rows, and with the box plan's strides (sy, sz) everything their stencil entries reference lies in three contiguous
// windows of x, [first - sy - 1, last + sy + 1] shifted by -sz, 0, +sz.  The CTA fetches its block tile (two bulk copies) and
// those three windows (three bulk copies, ~7 KB each) into shared memory and takes the operands from there; an entry outside
// the windows (the perturbation's added far columns, rows of a tile that spans more than the window holds) is gathered from
// global memory as before.  Nothing about the matrix is assumed: the windows are a cache, the column decides.
#include <algorithm>

#include "device_utils.cuh"
#include "spmv_internal.cuh"

namespace spmvb {

struct ExcArgs {
    const double *values;
    const int32_t *columns;
    const int32_t *rows;  // exception slot -> local row
    const double *x;
    double *y;
    int64_t x_col0, x_len;
    int64_t g0;  // x index of local row 0's own column: row_offset - x_col0
    int32_t width, e_begin, e_end, n_exc;
    int32_t sy;
    int64_t sz;
    int32_t cap;  // doubles per window (even)
};

#ifdef SPMVB_LAB  // measured slower than the ELL kernel with a row map (43 vs 34 us for the block of BASELINE config 4): lab builds only
template <int ROWS>
__global__ void __launch_bounds__(2 * ROWS) spmv_exception_window_kernel(ExcArgs p) {
    constexpr int THREADS = 2 * ROWS;
    extern __shared__ __align__(128) unsigned char smem[];
    const int w = p.width;
    double *sv = reinterpret_cast<double *>(smem);
    int32_t *sc = reinterpret_cast<int32_t *>(smem + (size_t)ROWS * w * 8);
    const uint32_t bytes_v = (uint32_t)ROWS * w * 8, bytes_c = (uint32_t)ROWS * w * 4;
    double *win = reinterpret_cast<double *>(smem + ((bytes_v + bytes_c + 127u) & ~127u));
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int32_t s_lo[3], s_len[3];  // windows in GLOBAL column numbers (int32, like the columns themselves)
    const int tile = p.e_begin / ROWS + blockIdx.x;
    const int e0 = tile * ROWS;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar[0]), 1);
        mbar_init(smem_u32(&bar[1]), 1);
        fence_mbar_init();
        // the block tile: contiguous, whole (the streams carry a tile of zeroed slack past n_exc)
        mbar_expect_tx(smem_u32(&bar[0]), bytes_v + bytes_c);
        bulk_g2s(smem_u32(sv), p.values + (int64_t)e0 * w, bytes_v, smem_u32(&bar[0]));
        bulk_g2s(smem_u32(sc), p.columns + (int64_t)e0 * w, bytes_c, smem_u32(&bar[0]));
        // the three windows of x around the tile's rows
        const int first = max(e0, p.e_begin), last = min(e0 + ROWS, p.e_end) - 1;
        const int64_t rlo = __ldg(p.rows + first) + p.g0, rhi = __ldg(p.rows + last) + p.g0;
        uint32_t total = 0;
        int64_t lo[3];
        int32_t len[3];
#pragma unroll
        for (int d = 0; d < 3; d++) {
            int64_t a = rlo + (d - 1) * p.sz - p.sy - 1, b = rhi + (d - 1) * p.sz + p.sy + 2;  // [a, b), x indices
            if (a < 0) a = 0;
            a &= ~(int64_t)1;  // 16-byte aligned start
            if (b > p.x_len) b = p.x_len;
            int64_t n = b > a ? ((b - a + 1) & ~(int64_t)1) : 0;  // whole 16-byte pieces
            if (n > p.cap) n = p.cap;
            if (a + n > p.x_len) n = (p.x_len - a) & ~(int64_t)1;  // never past the end of x
            const int64_t col = a + p.x_col0;                     // first global column of the window
            if (n < 0 || col < INT32_MIN || col + n > INT32_MAX) n = 0;  // no int32 column can lie in such a window
            lo[d] = a;
            len[d] = (int32_t)n;
            total += (uint32_t)len[d] * 8u;
        }
        mbar_expect_tx(smem_u32(&bar[1]), total);  // (0 bytes: the phase completes with this arrival)
#pragma unroll
        for (int d = 0; d < 3; d++) {
            s_lo[d] = len[d] > 0 ? (int32_t)(lo[d] + p.x_col0) : 0;
            s_len[d] = len[d];
            if (len[d] > 0) bulk_g2s(smem_u32(win + (size_t)d * p.cap), p.x + lo[d], (uint32_t)len[d] * 8u, smem_u32(&bar[1]));
        }
    }
    __syncthreads();  // barriers initialised, window bounds visible
    const int32_t lo0 = s_lo[0], lo1 = s_lo[1], lo2 = s_lo[2];
    const uint32_t n0 = (uint32_t)s_len[0], n1 = (uint32_t)s_len[1], n2 = (uint32_t)s_len[2];
    const int cap = p.cap;
    mbar_wait(smem_u32(&bar[0]), 0);
    mbar_wait(smem_u32(&bar[1]), 0);
    // Phase 1, all threads over the tile's ROWS x w entries (flat, conflict-free): the product v * x[c] replaces v.
    // inc/kernels.hpp:19-20: padding slots multiply 0.0 by x[own row] like any other entry.
    const int n_entries = ROWS * w;
    const double *__restrict__ x = p.x;
    const int64_t x_col0 = p.x_col0;
#pragma unroll 4
    for (int i = threadIdx.x; i < n_entries; i += THREADS) {
        const int32_t c = sc[i];
        const uint32_t o1 = (uint32_t)c - (uint32_t)lo1, o0 = (uint32_t)c - (uint32_t)lo0, o2 = (uint32_t)c - (uint32_t)lo2;  // wraps: in the window iff below its length
        double xv;
        if (o1 < n1) xv = win[cap + o1];
        else if (o0 < n0) xv = win[o0];
        else if (o2 < n2) xv = win[2 * cap + o2];
        else xv = __ldg(x + ((int64_t)c - x_col0));
        sv[i] = __dmul_rn(sv[i], xv);
    }
    __syncthreads();
    // Phase 2, a thread per row: the products summed in slot order (stride w doubles: conflict free for odd w)
    const int e = e0 + threadIdx.x;
    if (threadIdx.x < ROWS && e >= p.e_begin && e < p.e_end) {
        const double *pr = sv + threadIdx.x * w;
        double acc = 0.0;
        for (int k = 0; k < w; k++) acc = __dadd_rn(acc, pr[k]);
        p.y[__ldg(p.rows + e)] = acc;
    }
}

#endif  // SPMVB_LAB

// 0 launched, 1 not served (caller runs the ELL kernel with the row map), < 0 error
int launch_exception_window(const spmvb_matrix *a, const double *x, int64_t x_col0, int64_t x_len, double *y, int e_begin, int e_end,
                            cudaStream_t st) {
    if (e_end <= e_begin) return 0;
#ifndef SPMVB_LAB
    (void)a, (void)x, (void)x_col0, (void)x_len, (void)y, (void)st;
    return 1;  // the window kernels are compiled into lab builds only
#else
    // 0 auto = 1 the ELL kernel with a row map (measured faster on BASELINE config 4: 34 vs 43 us for the block), 32 / 64: this
    // kernel with that tile height
    const int mode = options().exception_kernel;
    if ((mode != 32 && mode != 64) || !a->box.valid || a->w_exc < 1 || a->w_exc > 64 || ((uintptr_t)x % 16) != 0) return 1;
    const int rows = mode == 32 ? 32 : 64;
    const auto &er = a->h_exc_rows;
    // window size: the tile's own span (1.3 x the average of this range) plus the stencil's reach either side
    const double gap = (double)(er[e_end - 1] - er[e_begin] + 1) / (double)(e_end - e_begin);
    const size_t block = ((size_t)rows * a->w_exc * 12 + 127) & ~(size_t)127;
    int64_t cap = (int64_t)(1.3 * gap * rows) + 2 * (int64_t)a->box.sy + 4;
    const int64_t cap_max = (int64_t)((100 * 1024 - block) / 24);
    cap = std::max<int64_t>(64, std::min(cap, cap_max)) & ~(int64_t)1;
    if (cap < 2 * (int64_t)a->box.sy + 4 + rows) return 1;  // lines too long for a window: nothing would be served from it
    const size_t smem = block + (size_t)cap * 24;
    ExcArgs p;
    p.values = static_cast<const double *>(a->s[SPMVB_S_EXC_VALUES]);
    p.columns = static_cast<const int32_t *>(a->s[SPMVB_S_EXC_COLUMNS]);
    p.rows = static_cast<const int32_t *>(a->s[SPMVB_S_EXC_ROWS]);
    p.x = x;
    p.y = y;
    p.x_col0 = x_col0;
    p.x_len = x_len;
    p.g0 = a->row_offset - x_col0;
    p.width = a->w_exc;
    p.e_begin = e_begin;
    p.e_end = e_end;
    p.n_exc = a->n_exc;
    p.sy = a->box.sy;
    p.sz = a->box.sz;
    p.cap = (int32_t)cap;
    const int t0 = e_begin / rows, nt = (e_end + rows - 1) / rows - t0;
    static PerDevice<bool> attr;
    if (!attr.get()) {
        if (cudaFuncSetAttribute(spmv_exception_window_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024) != cudaSuccess ||
            cudaFuncSetAttribute(spmv_exception_window_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024) != cudaSuccess)
            return -1;
        attr.get() = true;
    }
    if (rows == 32) spmv_exception_window_kernel<32><<<nt, 64, smem, st>>>(p);
    else spmv_exception_window_kernel<64><<<nt, 128, smem, st>>>(p);
    return check_launch("spmv_exception_window") == SPMVB_OK ? 0 : -1;
#endif
}

}  // namespace spmvb
