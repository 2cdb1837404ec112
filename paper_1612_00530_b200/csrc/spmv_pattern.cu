// Pattern-format SpMV (inc/compress.hpp:48-76; spmv: inc/kernels.hpp:25,35-36; PAPER.md:797-813
// List 1): production launchers, kernel selection, and the C-ABI SpMV entry points.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "pattern_kernels.cuh"
#include "spmv_internal.cuh"

namespace spmvb {

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
    if (neg1 && cp == 1) LAUNCH(true, 1); else LAUNCH(false, -1);  // the HPCG value pattern specialised; anything else: general variant
#undef LAUNCH
    return check_launch("spmv_pattern_box");
}

// v3 launch: returns 1 when the configuration / alignment is not served (caller falls back to v2)
template <int R, int WC, int Q, int LPS, int MINB, bool ALLV, int WA = 1, int LA = 0>
static int launch_box3(const spmvb_matrix *a, PatternArgs &p, cudaStream_t st) {
    const int64_t n_rows = (int64_t)p.row_end - p.row_begin;
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    const int n_planes = (int)((n_rows + sz - 1) / sz);
    const bool neg1 = p.v_off == -1.0;
    const int cp = a->box.center_pos;
    if (!ALLV && !(neg1 && cp == 1)) return 1;
    dim3 grid((p.sy + 64 * WA - 1) / (64 * WA), (p.plane_lines + R - 1) / R, (n_planes + (WC / WA) * Q - 1) / ((WC / WA) * Q));
    dim3 block(WC * 32);
#define LAUNCH3(NEG, CP) spmv_pattern_box3_kernel<R, WC, Q, LPS, MINB, NEG, CP, WA, LA><<<grid, block, 0, st>>>(p, n_planes)
    if constexpr (ALLV) {
        if (neg1 && cp == 1) LAUNCH3(true, 1); else LAUNCH3(false, -1);
    } else {
        LAUNCH3(true, 1);
    }
#undef LAUNCH3
    return check_launch("spmv_pattern_box3") == SPMVB_OK ? 0 : -1;
}

// Conditions of the v3 kernel: vector loads need even strides/offsets and 16-byte aligned
// arrays; all in-tile offsets must fit 32 bits; masks must fit the shared-memory table.
static bool box3_ok(const spmvb_matrix *a, const PatternArgs &p) {
    const int64_t sz = (int64_t)p.sy * p.plane_lines;
    return (p.sy % 2 == 0) && ((p.g0 + p.row_begin) % 2 == 0) && (p.row_begin % 2 == 0) &&
           ((uintptr_t)p.x % 16 == 0) && ((uintptr_t)p.y % 16 == 0) && ((uintptr_t)p.ids % 8 == 0) &&
           a->n_patterns <= kDictSmemPat && 6 * sz + 128 * (int64_t)p.sy + 4096 < INT32_MAX;
}

FusedDot *&fused_dot_request() {
    static thread_local FusedDot *req = nullptr;
    return req;
}

static int launch_pattern(const spmvb_matrix *a, const double *x, int64_t x_col0, int64_t x_len, double *y,
                          int row_begin, int row_end, cudaStream_t st) {
    // Hybrid handles: the exception block (below) shares nothing with the dictionary rows but x, and writes other rows of y;
    // it runs on the handle's second stream, forked here and joined at the end, so that the two kernels share the GPU.
    int e0 = 0, e1 = 0;
    if (a->n_exc > 0 && row_end > row_begin) {
        const auto &er = a->h_exc_rows;  // exception slots whose rows fall in [row_begin,row_end)
        e0 = (int)(std::lower_bound(er.begin(), er.end(), row_begin) - er.begin());
        e1 = (int)(std::lower_bound(er.begin(), er.end(), row_end) - er.begin());
    }
    const bool forked = e1 > e0 && options().exception_overlap != 0;
    if (forked) {
        if (!a->exc_stream) {
            SPMVB_CUDA(cudaStreamCreateWithFlags(&a->exc_stream, cudaStreamNonBlocking));
            for (auto &ev : a->exc_events) SPMVB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        }
        SPMVB_CUDA(cudaEventRecord(a->exc_events[0], st));
        SPMVB_CUDA(cudaStreamWaitEvent(a->exc_stream, a->exc_events[0], 0));
    }
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
        p.ids_avail = (int64_t)a->n - row_begin;
        p.sy = a->box.sy; p.plane_lines = a->box.valid ? a->box.sz / a->box.sy : 0;
        p.v_off = a->box.valid ? a->h_table[a->box.k_off] : 0.0;
        p.v_center = a->box.valid ? a->h_table[a->box.k_center] : 0.0;
        p.center_pos = a->box.center_pos;
        Options &o = options();
        p.prefetch = o.box_prefetch >= 0 ? o.box_prefetch : 2;
        p.prefetch_l1 = o.box_prefetch_l1;
        p.debug_nochain = kLabBuild ? o.debug_nochain : 0;
        if (FusedDot *req = fused_dot_request()) {  // x.y alongside y: every row through one ring launch, x[row] = the row's own entry
            if (a->n_exc == 0 && row_begin == 0 && row_end == a->n && a->row_offset == 0 && x_col0 == 0 && a->n_cols == a->n && x_len == a->n &&
                o.box_march == 0 && o.pattern_kernel == 0 && o.debug_nochain == 0) {
                p.dot_partial = req->partial;
                p.dot_capacity = req->capacity;
            }
        }
        const bool use_box = a->box.valid && o.pattern_kernel != 1;
        if (o.pattern_kernel == 2 && !a->box.valid)
            return fail(SPMVB_ERR_INVALID_ARGUMENT, "box kernel requested but the dictionary has no box plan");
        auto launch_list1 = [&]() -> int {  // List 1 as written: a thread per row, one round of gathers
            const int threads = 256;
            const int blocks = (row_end - row_begin + threads - 1) / threads;
            o.last_pattern_kernel = 1;
            const bool dict_smem = a->disp_total <= kDictSmemDisp && a->n_patterns <= kDictSmemPat && a->m <= kDictSmemTab;
            if (dict_smem) spmv_pattern_generic_kernel<true><<<blocks, threads, 0, st>>>(p);
            else spmv_pattern_generic_kernel<false><<<blocks, threads, 0, st>>>(p);
            return check_launch("spmv_pattern_generic");
        };
        bool done = false;
        if (use_box) {
            int rc3 = 1;  // 1 = not served by v3
            bool ring = false;
            // tensor-ring kernel (spmv_pattern_tma.cu): default for ranges of at least 8 planes; 90..94 force a variant
            const int64_t planes = ((int64_t)row_end - row_begin) / ((int64_t)p.sy * p.plane_lines);
            const bool want_ring = (o.box_march == 0 && planes >= 8) || (o.box_march >= 90 && o.box_march <= 120);
            if (o.pattern_kernel != 3 && want_ring && ring_ok(a, p)) {
                rc3 = launch_pattern_ring(o.box_march >= 90 ? o.box_march - 90 : 0, o.box_lines, a, p, st);
                if (rc3 < 0) return SPMVB_ERR_CUDA;
                ring = rc3 == 0;
            }
            // Short ranges the ring does not serve (lines narrower than a box, fewer than 8 planes -- a slab's boundary plane, a
            // 32^3 or 64^3 grid): the sliding-window kernels march a handful of long serial chains (15.7 us per SpMV at 32^3 and
            // 64^3 alike, graph-replayed); List 1 with a thread per row is one round of gathers: 4.0 / 6.7 us.  Above ~1 M rows the
            // windows win (7 vs 15.7 ns per 1000 rows).
            if (!ring && o.pattern_kernel == 0 && o.box_march == 0 && (int64_t)row_end - row_begin < (1 << 20)) {
                SPMVB_TRY(launch_list1());
                done = true;
            }
            if (!done && !ring && o.pattern_kernel != 3 && box3_ok(a, p)) {
                const int64_t n_planes = ((int64_t)row_end - row_begin + (int64_t)p.sy * p.plane_lines - 1) / ((int64_t)p.sy * p.plane_lines);
                if (n_planes == 1) {  // single-plane ranges (slab boundary planes): short marches, so that the plane fills the GPU
#ifdef SPMVB_LAB
                    if (o.box_lines == 16) rc3 = launch_box3<16, 4, 1, 2, 3, false>(a, p, st);
                    else if (o.box_lines == 8) rc3 = launch_box3<8, 4, 1, 2, 3, false>(a, p, st);
                    else if (o.box_lines == 2) rc3 = launch_box3<2, 4, 1, 2, 3, false>(a, p, st);
                    else
#endif
                    rc3 = launch_box3<4, 4, 1, 2, 3, false>(a, p, st);
                }
                else switch (o.box_march) {
#ifdef SPMVB_LAB
                    // measured alternatives kept selectable for A/B (profiles/r01_probe256_*.log, 256^3):
                    case 1: rc3 = launch_box3<16, 4, 2, 1, 3, false>(a, p, st); break;      // R=16 tiles            124 us
                    case 5: rc3 = launch_box3<16, 4, 1, 2, 3, false>(a, p, st); break;      // 1 plane, 2 lines/step 116-121 us
                    case 12: rc3 = launch_box3<16, 4, 2, 1, 3, false, 4>(a, p, st); break;  // CTA spans full lines  124 us
                    case 71: rc3 = launch_box3<8, 4, 2, 1, 4, false>(a, p, st); break;
                    case 72: rc3 = launch_box3<8, 4, 2, 1, 3, false, 1, 1>(a, p, st); break;
                    case 70: rc3 = launch_box3<8, 4, 2, 1, 2, false, 1, 1>(a, p, st); break;   // register look-ahead LA=1: 146 us (sweep: profiles/r01_probe256_lookahead_sweep.log)
                    case 20: case 30: case 35: case 47: case 62:                            // spmv_pattern_lab.cu
                        rc3 = launch_pattern_lab(o.box_march, a, p, st); break;
#endif
                    case 3: rc3 = launch_box3<8, 4, 2, 1, 3, true>(a, p, st); break;           // box3 default, forced
                    // <R=8 lines, 4 warps, Q=2 planes/thread, 1 line/step, 3 CTAs/SM>: 118-123 us
                    default: rc3 = launch_box3<8, 4, 2, 1, 3, true>(a, p, st); break;
                }
                if (rc3 < 0) return SPMVB_ERR_CUDA;
            }
            if (!done) o.last_pattern_kernel = rc3 == 1 ? 2 : (ring ? 9 : (o.box_march >= 20 && o.box_march < 70 ? 4 : 3));
            if (!done && rc3 == 1) {  // v2: any stride / alignment / value pattern
#ifdef SPMVB_LAB
                if (o.box_march == 11) SPMVB_TRY((launch_box_rw<32, 8, 1, 1>(a, p, st)));
                else
#endif
                SPMVB_TRY((launch_box_rw<16, 8, 2, 0>(a, p, st)));
            }
        } else {
            SPMVB_TRY(launch_list1());
        }
    }
    if (e1 > e0) {
        cudaStream_t se = forked ? a->exc_stream : st;
        const int rcw = launch_exception_window(a, x, x_col0, x_len, y, e0, e1, se);  // spmv_exception.cu
        if (rcw < 0) return SPMVB_ERR_CUDA;
        if (rcw == 1)
            SPMVB_TRY(launch_ell(static_cast<const double *>(a->s[SPMVB_S_EXC_VALUES]),
                                 static_cast<const int32_t *>(a->s[SPMVB_S_EXC_COLUMNS]), a->w_exc, x, x_col0, y, e0, e1,
                                 static_cast<const int32_t *>(a->s[SPMVB_S_EXC_ROWS]), se));
        if (forked) {
            SPMVB_CUDA(cudaEventRecord(a->exc_events[1], se));
            SPMVB_CUDA(cudaStreamWaitEvent(st, a->exc_events[1], 0));
        }
    }
    return SPMVB_OK;
}

}  // namespace spmvb

namespace spmvb {

// Pageable host vectors (a std::vector, a numpy array): a cudaMemcpy from pageable memory goes through the driver's own
// staging at ~7 GB/s per direction (19.5 ms per 256^3 SpMV against 3.2 ms from pinned buffers).  spmv_host stages them itself:
// process-wide pinned bounce buffers (grown on demand, kept), the copies in and out done by a few host threads, chunk by
// chunk inside the same three-stream pipeline, so that the memcpys, both PCIe directions and the kernels overlap.
struct HostStage {
    std::mutex lock;  // one staged call at a time (concurrent callers queue here; pinned callers never take it)
    double *x = nullptr, *y = nullptr;
    int64_t cap = 0;
    int ensure(int64_t n) {
        if (cap >= n) return SPMVB_OK;
        if (x) cudaFreeHost(x);
        if (y) cudaFreeHost(y);
        x = y = nullptr;
        cap = 0;
        if (cudaMallocHost(&x, (size_t)n * 8) != cudaSuccess || cudaMallocHost(&y, (size_t)n * 8) != cudaSuccess) {
            if (x) cudaFreeHost(x);
            x = y = nullptr;
            (void)cudaGetLastError();
            return SPMVB_ERR_NOMEM;
        }
        cap = n;
        return SPMVB_OK;
    }
};
static HostStage &host_stage() {
    static HostStage *s = new HostStage();  // never destroyed: the driver may be gone by the time statics are
    return *s;
}

static bool is_pageable(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

// dst[0,n) = src[0,n) by `threads` host threads (whole 4 KB blocks each)
static void parallel_copy(double *dst, const double *src, int64_t n, int threads) {
    if (n <= 0) return;
    if (threads <= 1 || n < (1 << 16)) {
        std::memcpy(dst, src, (size_t)n * 8);
        return;
    }
    const int64_t per = ((n + threads - 1) / threads + 511) / 512 * 512;
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; t++) {
        const int64_t b = t * per, e = std::min(n, b + per);
        if (b < e) pool.emplace_back([=] { std::memcpy(dst + b, src + b, (size_t)(e - b) * 8); });
    }
    std::memcpy(dst, src, (size_t)std::min(n, per) * 8);
    for (auto &th : pool) th.join();
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
    const int64_t n = a->n;
    // Reach of a row into x: known exactly for the pattern format (largest |displacement| of the dictionary,
    // no exception rows).  Then the call is pipelined over row chunks: while chunk c computes, x for the later
    // chunks is still arriving and y of the earlier chunks is already leaving (PCIe is full duplex).
    int64_t reach = -1;
    if (a->format == SPMVB_FMT_PATTERN && a->n_exc == 0 && n >= (1 << 20)) {
        reach = 0;
        for (int32_t d : a->h_disp_flat) reach = std::max<int64_t>(reach, d < 0 ? -(int64_t)d : d);
    }
    // pageable vectors go through pinned bounce buffers ("host_stage" = 0 leaves them to the driver)
    const bool stage_x = options().host_stage != 0 && n >= (1 << 18) && is_pageable(x_host);
    const bool stage_y = options().host_stage != 0 && n >= (1 << 18) && is_pageable(y_host);
    std::unique_lock<std::mutex> staged;
    const double *x_src = x_host;
    double *y_dst = y_host;
    const int copiers = std::max(1, std::min(options().host_copy_threads > 0 ? options().host_copy_threads : 8, (int)std::thread::hardware_concurrency()));
    if (stage_x || stage_y) {
        HostStage &hs = host_stage();
        staged = std::unique_lock<std::mutex>(hs.lock);
        if (hs.ensure(std::max<int64_t>(x_len, n)) != SPMVB_OK) {
            staged.unlock();  // no pinned memory to be had: the driver's pageable copies
        } else {
            if (stage_x) x_src = hs.x;
            if (stage_y) y_dst = hs.y;
        }
    }
    const bool sx = x_src != x_host, sy_ = y_dst != y_host;
    if (reach < 0 || reach * 8 > n) {  // plain path: copy, run, copy
        if (sx) parallel_copy(const_cast<double *>(x_src), x_host, x_len, copiers);
        SPMVB_CUDA(cudaMemcpyAsync(a->scratch_x, x_src, (size_t)x_len * 8, cudaMemcpyHostToDevice, nullptr));
        SPMVB_TRY(spmvb_spmv(a, a->scratch_x, 0, x_len, a->scratch_y, 0, a->n, nullptr));
        SPMVB_CUDA(cudaMemcpyAsync(y_dst, a->scratch_y, (size_t)a->n * 8, cudaMemcpyDeviceToHost, nullptr));
        SPMVB_CUDA(cudaStreamSynchronize(nullptr));
        if (sy_) parallel_copy(y_host, y_dst, n, copiers);
        return SPMVB_OK;
    }
    constexpr int kMaxChunks = 64;
    const int kChunks = std::min(kMaxChunks, options().host_chunks > 0 ? options().host_chunks : 8);
    if (!a->pipe_streams[0]) {
        for (int i = 0; i < 3; i++) SPMVB_CUDA(cudaStreamCreateWithFlags(&a->pipe_streams[i], cudaStreamNonBlocking));
        for (int i = 0; i < 2 * kMaxChunks; i++) SPMVB_CUDA(cudaEventCreateWithFlags(&a->pipe_events[i], cudaEventDisableTiming));
    }
    cudaStream_t s_in = a->pipe_streams[0], s_run = a->pipe_streams[1], s_out = a->pipe_streams[2];
    // chunk boundaries on whole planes of the box plan when there is one (tiles then stay aligned), multiples of 4 rows otherwise
    const int64_t unit = a->box.valid ? (int64_t)a->box.sz : 4;
    const int64_t units = (n + unit - 1) / unit;
    const int64_t per = std::max<int64_t>(1, (units + kChunks - 1) / kChunks) * unit;
    // staged y: a drain thread copies each chunk out of the bounce buffer as soon as its D2H has landed (one event per chunk)
    std::vector<int64_t> bounds;
    for (int64_t r0 = 0; r0 < n; r0 += per) bounds.push_back(r0);
    bounds.push_back(n);
    const int n_chunks = (int)bounds.size() - 1;
    if (sy_ && !a->pipe_out_events[0])
        for (auto &ev : a->pipe_out_events) SPMVB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    std::thread drain;
    int queued = 0;          // chunks whose D2H has been enqueued (read by the drain thread through `queued_pub`)
    std::atomic<int> queued_pub{0};
    std::atomic<bool> failed{false};
    if (sy_)
        drain = std::thread([&] {
            cudaSetDevice(a->device);  // a new host thread starts on device 0
            for (int k = 0; k < n_chunks; k++) {
                while (queued_pub.load(std::memory_order_acquire) <= k && !failed.load()) std::this_thread::yield();
                if (failed.load()) return;
                if (cudaEventSynchronize(a->pipe_out_events[k]) != cudaSuccess) {
                    failed.store(true);
                    return;
                }
                parallel_copy(y_host + bounds[k], y_dst + bounds[k], bounds[k + 1] - bounds[k], std::max(1, copiers / 2));
            }
        });
    auto bail = [&](int code) {
        failed.store(true);
        if (drain.joinable()) drain.join();
        return code;
    };
    int64_t sent = 0;
    for (int c = 0; c < n_chunks; c++) {
        const int64_t r0 = bounds[c], r1 = bounds[c + 1];
        // whole 4 KB blocks: a copy that starts at an odd element runs at 80 % of the PCIe rate (tests/e2e_probe.py)
        const int64_t need = std::min(n, (r1 + reach + 511) / 512 * 512);
        if (need > sent) {
            if (sx) parallel_copy(const_cast<double *>(x_src) + sent, x_host + sent, need - sent, sy_ ? std::max(1, copiers / 2) : copiers);
            if (cudaMemcpyAsync(a->scratch_x + sent, x_src + sent, (size_t)(need - sent) * 8, cudaMemcpyHostToDevice, s_in) != cudaSuccess)
                return bail(fail(SPMVB_ERR_CUDA, "spmv_host: %s", cudaGetErrorString(cudaGetLastError())));
            sent = need;
        }
        bool ok = cudaEventRecord(a->pipe_events[2 * c], s_in) == cudaSuccess && cudaStreamWaitEvent(s_run, a->pipe_events[2 * c], 0) == cudaSuccess;
        if (ok && spmvb_spmv(a, a->scratch_x, 0, x_len, a->scratch_y, (int32_t)r0, (int32_t)r1, s_run) != SPMVB_OK) return bail(SPMVB_ERR_CUDA);
        ok = ok && cudaEventRecord(a->pipe_events[2 * c + 1], s_run) == cudaSuccess && cudaStreamWaitEvent(s_out, a->pipe_events[2 * c + 1], 0) == cudaSuccess &&
             cudaMemcpyAsync(y_dst + r0, a->scratch_y + r0, (size_t)(r1 - r0) * 8, cudaMemcpyDeviceToHost, s_out) == cudaSuccess;
        if (ok && sy_) ok = cudaEventRecord(a->pipe_out_events[c], s_out) == cudaSuccess;
        if (!ok) return bail(fail(SPMVB_ERR_CUDA, "spmv_host: %s", cudaGetErrorString(cudaGetLastError())));
        queued = c + 1;
        queued_pub.store(queued, std::memory_order_release);
    }
    if (drain.joinable()) drain.join();
    if (failed.load()) return fail(SPMVB_ERR_CUDA, "spmv_host: a copy failed: %s", cudaGetErrorString(cudaGetLastError()));
    SPMVB_CUDA(cudaStreamSynchronize(s_out));
    return SPMVB_OK;
}

}  // extern "C"
