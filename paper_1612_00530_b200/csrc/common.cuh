// Internal declarations shared by the translation units of libspmvcomp_b200.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "spmvcomp_b200.h"

namespace spmvb {

// ---- error plumbing ---------------------------------------------------------
std::string &last_error_ref();
int fail(int code, const char *fmt, ...);

#define SPMVB_CUDA(expr)                                                                   \
    do {                                                                                   \
        cudaError_t e__ = (expr);                                                          \
        if (e__ != cudaSuccess)                                                            \
            return ::spmvb::fail(SPMVB_ERR_CUDA, "%s failed: %s (%s:%d)", #expr,           \
                                 cudaGetErrorString(e__), __FILE__, __LINE__);             \
    } while (0)

#define SPMVB_TRY(expr)              \
    do {                             \
        int rc__ = (expr);           \
        if (rc__ != SPMVB_OK) return rc__; \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Per-device "done once" state (function attributes and occupancy are properties of a kernel *on a device*;
// a process may drive several devices through spmvb_set_device).
constexpr int kMaxDevices = 64;
inline int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
    return d;
}
template <typename T>
struct PerDevice {
    T v[kMaxDevices] = {};
    T &get() { return v[current_device()]; }
};

// Measured experiments and ablations (spmv_pattern_lab.cu, the non-default instantiations selected by "box_march" /
// "ell_kernel" / "debug_nochain") are compiled only with -DSPMVB_LAB (make LAB=1 -> libspmvcomp_b200_lab.so); some of
// them skip work on purpose and return wrong y.  The default library cannot reach any of them.
#ifdef SPMVB_LAB
constexpr bool kLabBuild = true;
#else
constexpr bool kLabBuild = false;
#endif

// SMs of the current device (grids are sized in multiples of it).
inline int sm_count() {
    static PerDevice<int> n;
    int &v = n.get();
    if (v == 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 1;
    }
    return v;
}

// Rows per CTA tile of the row-major ELL-like streams.  Device allocations of
// those streams are padded to a whole number of tiles so a tile can always be
// fetched with full 16-byte vector loads.
constexpr int kTileRows = 128;

// Sliding-window ("box") plan for a pattern dictionary whose dominant pattern is a
// 3x3x3 box of displacements dx + sy*dy + sz*dz (the 27-point stencil in x-fastest
// numbering), all 26 off-centre entries sharing one table value.
struct BoxPlan {
    bool valid = false;
    int32_t sy = 0, sz = 0;     // strides found in the dictionary
    int32_t center_pos = 0;     // 0 centre first, 1 centre last, 2 centre in place (m == 1)
    int32_t k_off = 0, k_center = 0;  // value-table indices
    std::vector<uint32_t> masks;      // per pattern: 27-bit sub-box mask, or kGenericMask
};
constexpr uint32_t kGenericMask = 0xFFFFFFFFu;

}  // namespace spmvb

struct SymgsGraph {  // the recorded launches of one symgs sweep (symgs.cu)
    cudaGraphExec_t exec = nullptr;
    cudaStream_t capture_stream = nullptr;
    const double *b = nullptr;
    double *x = nullptr;
    int nx = 0, ny = 0, nz = 0;
};

struct spmvb_matrix {
    int32_t format = 0;
    int32_t device = 0;
    int32_t n = 0, width = 0, m = 0, n_patterns = 0, n_exc = 0, w_exc = 0, values_in_pattern = 0;
    int64_t nnz = 0, row_offset = 0, disp_total = 0, n_cols = 0;
    int64_t col_min = 0, col_max = -1;  // pattern handles: range of global columns the rows reference (col_max < col_min: unknown)
    void *s[SPMVB_S_COUNT_] = {};
    uint64_t bytes[SPMVB_S_COUNT_] = {};
    // host mirrors of the small pattern-side tables
    std::vector<double> h_table;
    std::vector<int64_t> h_disp_offsets;
    std::vector<int32_t> h_disp_flat, h_ends_flat, h_exc_rows;
    std::vector<int32_t> h_first_rows;  // first local row of each pattern (device-built handles)
    // persistent scratch of spmvb_spmv_host (x and y on the device)
    mutable double *scratch_x = nullptr, *scratch_y = nullptr;
    mutable int64_t scratch_x_len = 0;
    // work vectors of spmvb_cg_solve (r, p, Ap: 3n doubles), kept between solves on this handle unless "cg_keep_workspace" is 0
    mutable double *cg_ws = nullptr;
    mutable int cg_ws_busy = 0;  // taken with an atomic exchange: a second concurrent solve on the handle allocates its own
    mutable SymgsGraph symgs_graph;
    mutable uint32_t *symgs_mask = nullptr;    // CSR handles: per row, which of the 27 box positions its entries occupy (symgs.cu, the pipelined sweep)
    mutable int symgs_box[3] = {0, 0, 0};      // ... the grid it was derived for; symgs_box_ok: every row is a sub-box of its node's 27 neighbours
    mutable int symgs_box_ok = 0;
    mutable int symgs_checked[3] = {0, 0, 0};  // CSR handles: grid whose hyperplane schedule was verified against the matrix (symgs.cu)
    // streams / events of the pipelined host-buffer SpMV (created on first use)
    mutable cudaStream_t pipe_streams[3] = {};
    mutable cudaEvent_t pipe_events[128] = {};
    mutable cudaEvent_t pipe_out_events[64] = {};  // staged (pageable) y: one per chunk, the drain thread waits on them
    mutable cudaStream_t exc_stream = nullptr;  // hybrid handles: the exception block runs beside the dictionary rows (spmv_pattern.cu)
    mutable cudaEvent_t exc_events[2] = {};
    spmvb::BoxPlan box;
    uint32_t *d_masks = nullptr;      // device copy of box.masks
    int32_t *d_disp_off32 = nullptr;  // 32-bit copy of disp_offsets for the kernels
};

namespace spmvb {

// Allocates `bytes` (+ zeroed slack so vector loads of a partial tile stay in bounds).
int dev_alloc(spmvb_matrix *a, int sid, uint64_t bytes, uint64_t slack = 0);
int upload_stream(spmvb_matrix *a, int sid, const void *host, uint64_t bytes, uint64_t slack = 0);
int finish_pattern_handle(spmvb_matrix *a);  // builds host mirrors' device copies and the box plan
void analyse_box_plan(spmvb_matrix *a);
void destroy(spmvb_matrix *a);

struct Options {
    int pattern_kernel = 0;  // 0 auto, 1 generic (List 1), 2 box (v3, else v2), 3 box v2 only
    int ell_kernel = 0;      // 0 auto (ELL: TMA bulk pipeline, vt: staged), 1 naive, 2 staged vector loads, 3 TMA for vt too
    int box_march = 0;       // 0 default
    int box_prefetch = -1;   // L2 prefetch distance in lines (-1 = default)
    int box_prefetch_l1 = 0; // L1 prefetch distance in lines (0 = off)
    int debug_nochain = 0;   // measurement only
    int box_lines = 0;       // lines per CTA march of the tensor-ring kernel (0 = default)
    int exception_carveout = 0; // hybrid format, exception block kernel: preferred shared-memory carve-out in percent (0 = default 60, -1 = the driver's choice): less shared memory = fewer CTAs per SM and more L1 for the scattered gathers
    int exception_overlap = 1; // hybrid format: 1 the exception block on a second stream beside the dictionary rows (fork / join by events), 0 one after the other
    int exception_kernel = 0; // hybrid format, exception rows: 0 / 1 the ELL kernel with a row map (all gathers of a row in one batch), 64 / 32 shared-memory windows of x with that tile height
    int ring_min_steps = 0;  // tensor ring: fewest line steps per chunk before the grid shrinks below a full wave (0 = default 4)
    int ring_two_lines = 1;  // tensor ring, x far beyond L2 and strips in fours: two lines per step (0: one, as everywhere else)
    int ring_pdl = 1;        // tensor ring launched with programmatic stream serialization (its preamble overlaps the previous kernel's tail)
    int ring_leftover = 0;   // tensor ring, left-over column (64 | sy): 0 summed by the last strip's warp from its ring, 1 row by row after the marches
    int slab_graph = 1;         // 1: spmvb_slab_spmv records its exchange copies and launches into a CUDA graph and replays it
    int symgs_lag = 0;          // pipelined sweep: steps a plane trails its predecessor by (>= 7; 0 = 7)
    int symgs_pipeline = 1;     // 1: matrices whose rows are sub-boxes of the 27-point stencil are swept by the plane-per-CTA pipeline; 0: never
    int symgs_persistent = 1;   // 1: a symgs sweep is one cooperative launch that walks the levels itself (grid-wide barriers); 0: a launch per level
    int symgs_graph = 1;        // 1: a symgs sweep's launches are recorded into a CUDA graph and replayed
    int cg_fused_scalars = 1;   // cg_solve's vector kernel: 1 beta / stop flag / record by its last block (4 launches per iteration); 2 also alpha, formed at its head by every block (3 launches); 0 separate alpha and beta kernels (5 launches)
    int cg_pdl = 0;             // 1: the fused vector kernel and the direction kernel are launched with programmatic stream serialization (measured: no gain inside the replayed graph)
    int cg_graph = 1;           // 1: cg_solve records its iteration into a CUDA graph after the first and replays it
    int last_symgs_kernel = 0;  // read-only: what swept last: 0 a launch per level (or their graph), 1 the grid-barrier kernel, 2 the plane pipeline
    int last_cg_graph = 0;      // read-only: 1 when the last cg_solve replayed a graph
    int cg_fused_dot = 1;       // 1: cg_solve takes p.Ap from the SpMV kernel where that kernel offers it (pattern format, tensor ring)
    int last_cg_fused_dot = 0;  // read-only: 1 when the last iteration of the last cg_solve took p.Ap from the SpMV kernel
    int cg_keep_workspace = 1;  // 1: spmvb_cg_solve keeps its 3n work doubles on the handle until spmvb_free
    int host_stage = 1;      // spmv_host: 1 pageable host vectors go through pinned bounce buffers filled / drained by host threads; 0 the driver's pageable copies
    int host_copy_threads = 0; // ... that many copier threads (0 = default 8, at most the host's hardware threads)
    int host_chunks = 0;     // row chunks of the pipelined host-buffer SpMV (0 = default 8, at most 64)
    int last_pattern_kernel = 0;  // read-only: kernel family of the last pattern launch (1 List 1, 2 box v2, 3 box3, 4 lab, 9 tensor ring)
};
Options &options();  // per host thread

}  // namespace spmvb
