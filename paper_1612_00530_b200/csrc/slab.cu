// z-slab SpMV behind the C-ABI (SURVEY 8b "spmv_multi", 8e; the row ranges of unchecked::spmv_rows,
// inc/kernels.hpp:27-36; the paper's distribution of the grid over processes).
//
// A slab owns planes [z0, z1) of the global grid = a contiguous row range.  Its local vector is
//     x_ghosted = [ghost plane | owned planes | ghost plane]        (x_col0 = row_offset - plane, x_len = n + 2 plane)
// and per SpMV the first / last owned plane of each neighbour lands in the ghost planes.
//
//   spmvb_slab_*   one slab: the exchange as copies from the neighbours' planes (peer-mapped or same-device pointers) and
//                  the SpMV, recorded once into a CUDA graph and replayed; or the two halves (interior / boundary planes)
//                  for callers that run the exchange themselves (NCCL send/recv on their own stream).
//   spmvb_multi_*  one host thread driving G slabs on a device list (devices may repeat: logical slabs on one device):
//                  device-side build per slab, dictionary merge, seeded x, SpMV with exchange, timing, download.
//
// Schedules (spmvb_slab_mode), measured in tests/slab_probe.py:
//   SERIAL   ghost copies, then ONE launch over all owned planes (the tensor-ring kernel at full size).  The exchange
//            latency is exposed, the decomposition costs nothing else.
//   OVERLAP  ghost copies on a side stream while the planes that need no ghost are computed; the first and last owned
//            plane follow (two short launches on two streams).  Hides a slow exchange at the price of the short launches.
#include <algorithm>
#include <chrono>
#include <map>
#include <memory>
#include <vector>

#include "common.cuh"

using namespace spmvb;

struct spmvb_slab {
    const spmvb_matrix *a = nullptr;
    int device = 0;
    int64_t plane = 0;
    int has_lower = 0, has_upper = 0;
    cudaStream_t side = nullptr, capture = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_copied = nullptr, ev_side_done = nullptr;
    // the recorded SpMV (exchange + launches) for one set of pointers
    struct Key {
        const double *x = nullptr, *lo = nullptr, *hi = nullptr;
        double *y = nullptr;
        int mode = -1;
        bool operator==(const Key &o) const { return x == o.x && y == o.y && lo == o.lo && hi == o.hi && mode == o.mode; }
    } key, seen;
    cudaGraphExec_t exec = nullptr;
    int last_was_graph = 0;
};

namespace {

struct DeviceScope {  // a slab lives on its own device; restore the caller's on the way out
    int prev = -1;
    explicit DeviceScope(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

int ghost_copies(const spmvb_slab *s, double *x, const double *lo, const double *hi, cudaStream_t st) {
    const size_t bytes = (size_t)s->plane * 8;
    // cudaMemcpyDefault: same-device and peer-mapped sources alike (unified addressing resolves the route)
    if (lo && s->has_lower) SPMVB_CUDA(cudaMemcpyAsync(x, lo, bytes, cudaMemcpyDefault, st));
    if (hi && s->has_upper) SPMVB_CUDA(cudaMemcpyAsync(x + s->plane + s->a->n, hi, bytes, cudaMemcpyDefault, st));
    return SPMVB_OK;
}

// rows [0, lo_rows) need the lower ghost plane, rows [hi_rows, n) the upper one
void split_rows(const spmvb_slab *s, int32_t *lo_rows, int32_t *hi_rows) {
    const int64_t n = s->a->n;
    const int64_t lo = s->has_lower ? std::min<int64_t>(s->plane, n) : 0;
    const int64_t hi = s->has_upper ? std::max<int64_t>(n - s->plane, lo) : n;
    *lo_rows = (int32_t)lo;
    *hi_rows = (int32_t)hi;
}

int run_rows(const spmvb_slab *s, const double *x, double *y, int32_t b, int32_t e, cudaStream_t st) {
    if (e <= b) return SPMVB_OK;
    return spmvb_spmv(s->a, x, s->a->row_offset - s->plane, (int64_t)s->a->n + 2 * s->plane, y, b, e, st);
}

int enqueue(spmvb_slab *s, double *x, double *y, const double *lo, const double *hi, int mode, cudaStream_t st) {
    const bool exchange = (lo && s->has_lower) || (hi && s->has_upper);
    if (mode == SPMVB_SLAB_SERIAL || !(s->has_lower || s->has_upper)) {
        SPMVB_TRY(ghost_copies(s, x, lo, hi, st));
        return run_rows(s, x, y, 0, s->a->n, st);
    }
    int32_t lo_rows, hi_rows;
    split_rows(s, &lo_rows, &hi_rows);
    SPMVB_CUDA(cudaEventRecord(s->ev_fork, st));  // x is ready
    SPMVB_CUDA(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
    if (exchange) SPMVB_TRY(ghost_copies(s, x, lo, hi, s->side));
    SPMVB_CUDA(cudaEventRecord(s->ev_copied, s->side));
    SPMVB_TRY(run_rows(s, x, y, lo_rows, hi_rows, st));        // planes that need no ghost, while the copies run
    SPMVB_TRY(run_rows(s, x, y, 0, lo_rows, s->side));         // first owned plane, behind the copies on the side stream
    SPMVB_CUDA(cudaEventRecord(s->ev_side_done, s->side));
    SPMVB_CUDA(cudaStreamWaitEvent(st, s->ev_copied, 0));
    SPMVB_TRY(run_rows(s, x, y, hi_rows, s->a->n, st));        // last owned plane: the two share the GPU once the interior drains
    SPMVB_CUDA(cudaStreamWaitEvent(st, s->ev_side_done, 0));
    return SPMVB_OK;
}

}  // namespace

extern "C" {

int spmvb_slab_create(const spmvb_matrix *a, int64_t plane_rows, int32_t has_lower, int32_t has_upper, spmvb_slab **out) {
    if (!out) return fail(SPMVB_ERR_INVALID_ARGUMENT, "slab_create: out is NULL");
    *out = nullptr;
    if (!a || plane_rows < 1 || (a->format != SPMVB_FMT_ELL && a->format != SPMVB_FMT_VT && a->format != SPMVB_FMT_PATTERN))
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "slab_create: needs an ELL / vt / pattern handle and a plane of >= 1 rows");
    if (a->n % plane_rows != 0 || a->row_offset % plane_rows != 0)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "slab_create: %d rows at offset %lld are not whole planes of %lld rows", a->n,
                    (long long)a->row_offset, (long long)plane_rows);
    // Only the one-plane halo travels: every column the rows reference must lie in [row_offset - plane, row_offset + n + plane).
    // (Known for pattern handles; e.g. the perturbed grid of BASELINE config 4 adds entries at random columns and cannot be cut.)
    if (a->format == SPMVB_FMT_PATTERN && a->col_max >= a->col_min &&
        (a->col_min < a->row_offset - plane_rows || a->col_max >= a->row_offset + a->n + plane_rows))
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "slab_create: rows reference columns [%lld, %lld], beyond the one-plane halo of rows [%lld, %lld)",
                    (long long)a->col_min, (long long)a->col_max, (long long)a->row_offset, (long long)(a->row_offset + a->n));
    auto s = std::make_unique<spmvb_slab>();
    s->a = a;
    s->device = a->device;
    s->plane = plane_rows;
    s->has_lower = has_lower != 0;
    s->has_upper = has_upper != 0;
    DeviceScope scope(s->device);
    SPMVB_CUDA(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
    SPMVB_CUDA(cudaStreamCreateWithFlags(&s->capture, cudaStreamNonBlocking));
    SPMVB_CUDA(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
    SPMVB_CUDA(cudaEventCreateWithFlags(&s->ev_copied, cudaEventDisableTiming));
    SPMVB_CUDA(cudaEventCreateWithFlags(&s->ev_side_done, cudaEventDisableTiming));
    *out = s.release();
    return SPMVB_OK;
}

int spmvb_slab_destroy(spmvb_slab *s) {
    if (!s) return SPMVB_OK;
    DeviceScope scope(s->device);
    if (s->exec) cudaGraphExecDestroy(s->exec);
    if (s->side) cudaStreamDestroy(s->side);
    if (s->capture) cudaStreamDestroy(s->capture);
    for (cudaEvent_t e : {s->ev_fork, s->ev_copied, s->ev_side_done})
        if (e) cudaEventDestroy(e);
    delete s;
    return SPMVB_OK;
}

int spmvb_slab_spmv(spmvb_slab *s, double *x_ghosted, double *y, const double *lower_src, const double *upper_src, int32_t mode,
                    void *stream) {
    if (!s || !x_ghosted || !y) return fail(SPMVB_ERR_INVALID_ARGUMENT, "slab_spmv: NULL argument");
    if (mode != SPMVB_SLAB_SERIAL && mode != SPMVB_SLAB_OVERLAP) return fail(SPMVB_ERR_INVALID_ARGUMENT, "slab_spmv: unknown mode %d", mode);
    DeviceScope scope(s->device);
    cudaStream_t st = as_stream(stream);
    const spmvb_slab::Key k{x_ghosted, lower_src, upper_src, y, mode};
    s->last_was_graph = 0;
    if (!options().slab_graph) return enqueue(s, x_ghosted, y, lower_src, upper_src, mode, st);
    if (s->exec && s->key == k) {
        SPMVB_CUDA(cudaGraphLaunch(s->exec, st));
        s->last_was_graph = 1;
        return SPMVB_OK;
    }
    // First call with these pointers: direct launches (they also complete every lazy set-up of the kernels).  Second call:
    // the same sequence is recorded into a graph -- copies, launches and the fork / join of the side stream -- and from
    // then on a SpMV is one graph launch on the host.
    if (!(s->seen == k)) {
        s->seen = k;
        return enqueue(s, x_ghosted, y, lower_src, upper_src, mode, st);
    }
    if (s->exec) {
        cudaGraphExecDestroy(s->exec);
        s->exec = nullptr;
    }
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(s->capture, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
        const int rc = enqueue(s, x_ghosted, y, lower_src, upper_src, mode, s->capture);
        const bool ended = cudaStreamEndCapture(s->capture, &graph) == cudaSuccess && graph;
        if (rc != SPMVB_OK || !ended || cudaGraphInstantiate(&s->exec, graph, nullptr, nullptr, 0) != cudaSuccess) s->exec = nullptr;
        if (graph) cudaGraphDestroy(graph);
    }
    (void)cudaGetLastError();  // a failed capture leaves the direct launches
    if (!s->exec) return enqueue(s, x_ghosted, y, lower_src, upper_src, mode, st);
    s->key = k;
    SPMVB_CUDA(cudaGraphLaunch(s->exec, st));
    s->last_was_graph = 1;
    return SPMVB_OK;
}

int spmvb_slab_interior(spmvb_slab *s, const double *x_ghosted, double *y, void *stream) {
    if (!s || !x_ghosted || !y) return fail(SPMVB_ERR_INVALID_ARGUMENT, "slab_interior: NULL argument");
    DeviceScope scope(s->device);
    int32_t lo_rows, hi_rows;
    split_rows(s, &lo_rows, &hi_rows);
    return run_rows(s, x_ghosted, y, lo_rows, hi_rows, as_stream(stream));
}

int spmvb_slab_boundary(spmvb_slab *s, const double *x_ghosted, double *y, void *stream) {
    if (!s || !x_ghosted || !y) return fail(SPMVB_ERR_INVALID_ARGUMENT, "slab_boundary: NULL argument");
    DeviceScope scope(s->device);
    cudaStream_t st = as_stream(stream);
    int32_t lo_rows, hi_rows;
    split_rows(s, &lo_rows, &hi_rows);
    if (lo_rows > 0 && hi_rows < s->a->n) {  // two independent planes: side by side on two streams
        SPMVB_CUDA(cudaEventRecord(s->ev_fork, st));
        SPMVB_CUDA(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
        SPMVB_TRY(run_rows(s, x_ghosted, y, 0, lo_rows, s->side));
        SPMVB_CUDA(cudaEventRecord(s->ev_side_done, s->side));
        SPMVB_TRY(run_rows(s, x_ghosted, y, hi_rows, s->a->n, st));
        SPMVB_CUDA(cudaStreamWaitEvent(st, s->ev_side_done, 0));
        return SPMVB_OK;
    }
    SPMVB_TRY(run_rows(s, x_ghosted, y, 0, lo_rows, st));
    return run_rows(s, x_ghosted, y, hi_rows, s->a->n, st);
}

int spmvb_slab_last_was_graph(const spmvb_slab *s, int32_t *flag) {
    if (!s || !flag) return fail(SPMVB_ERR_INVALID_ARGUMENT, "NULL argument");
    *flag = s->last_was_graph;
    return SPMVB_OK;
}

// ---- peer memory across processes (one process per GPU): CUDA IPC handles of cudaMalloc'ed vectors ----------------
int spmvb_ipc_export(const void *dev_base, unsigned char handle[64]) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    if (!dev_base || !handle) return fail(SPMVB_ERR_INVALID_ARGUMENT, "ipc_export: NULL argument");
    cudaIpcMemHandle_t h;
    SPMVB_CUDA(cudaIpcGetMemHandle(&h, const_cast<void *>(dev_base)));
    memcpy(handle, &h, 64);
    return SPMVB_OK;
}

int spmvb_ipc_open(const unsigned char handle[64], void **dev_ptr) {
    if (!handle || !dev_ptr) return fail(SPMVB_ERR_INVALID_ARGUMENT, "ipc_open: NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    SPMVB_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return SPMVB_OK;
}

int spmvb_ipc_close(void *dev_ptr) {
    if (dev_ptr) SPMVB_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return SPMVB_OK;
}

}  // extern "C"

// =====================================================================================================================
// spmvb_multi: G slabs driven by one host thread
// =====================================================================================================================
struct spmvb_multi {
    struct Part {
        int device = 0;
        int64_t z0 = 0, z1 = 0;
        spmvb_matrix *a = nullptr;
        spmvb_slab *slab = nullptr;
        double *x = nullptr, *y = nullptr;  // x ghosted
        cudaStream_t st = nullptr;
        cudaEvent_t t0 = nullptr, t1 = nullptr;
    };
    spmvb_grid grid{};
    int32_t format = SPMVB_FMT_PATTERN;
    int64_t plane = 0;
    std::vector<Part> parts;
};

namespace {

void multi_free(spmvb_multi *m) {
    if (!m) return;
    for (auto &p : m->parts) {
        DeviceScope scope(p.device);
        if (p.slab) spmvb_slab_destroy(p.slab);
        if (p.a) spmvb_matrix_destroy(p.a);
        if (p.x) cudaFree(p.x);
        if (p.y) cudaFree(p.y);
        if (p.st) cudaStreamDestroy(p.st);
        if (p.t0) cudaEventDestroy(p.t0);
        if (p.t1) cudaEventDestroy(p.t1);
    }
    delete m;
}

// Per-slab dictionaries -> the numbering a single-matrix compression issues: ids by first occurrence in ascending GLOBAL
// row order (the C++ twin of slab.py:merge_dictionaries).  Rewrites every part's dictionary and ids.
int merge_dictionaries(spmvb_multi *m) {
    using Shape = std::pair<std::vector<int32_t>, std::vector<int32_t>>;  // (displacements, ends)
    std::map<Shape, int64_t> first_of;
    std::vector<std::vector<Shape>> shapes(m->parts.size());
    int mt = -1;
    for (size_t g = 0; g < m->parts.size(); g++) {
        const spmvb_matrix *a = m->parts[g].a;
        if (mt < 0) mt = a->m;
        if (a->m != mt || (g > 0 && a->h_table != m->parts[0].a->h_table)) return fail(SPMVB_ERR_INTEGRITY, "slabs disagree on the value table");
        std::vector<int32_t> first(std::max(a->n_patterns, 1));
        SPMVB_TRY(spmvb_pattern_first_rows(a, first.data()));
        for (int p = 0; p < a->n_patterns; p++) {
            Shape sh{std::vector<int32_t>(a->h_disp_flat.begin() + a->h_disp_offsets[p], a->h_disp_flat.begin() + a->h_disp_offsets[p + 1]),
                     std::vector<int32_t>(a->h_ends_flat.begin() + (size_t)p * a->m, a->h_ends_flat.begin() + (size_t)(p + 1) * a->m)};
            const int64_t fr = a->row_offset + first[p];
            auto it = first_of.find(sh);
            if (it == first_of.end() || fr < it->second) first_of[sh] = fr;
            shapes[g].push_back(std::move(sh));
        }
    }
    std::vector<std::pair<int64_t, const Shape *>> order;
    for (auto &kv : first_of) order.push_back({kv.second, &kv.first});
    std::sort(order.begin(), order.end(), [](auto &l, auto &r) { return l.first < r.first; });
    std::map<Shape, int32_t> new_id;
    std::vector<int64_t> offs(1, 0);
    std::vector<int32_t> flat, ends;
    for (size_t i = 0; i < order.size(); i++) {
        new_id[*order[i].second] = (int32_t)i;
        flat.insert(flat.end(), order[i].second->first.begin(), order[i].second->first.end());
        ends.insert(ends.end(), order[i].second->second.begin(), order[i].second->second.end());
        offs.push_back((int64_t)flat.size());
    }
    for (size_t g = 0; g < m->parts.size(); g++) {
        auto &p = m->parts[g];
        std::vector<int32_t> map(std::max<size_t>(shapes[g].size(), 1));
        for (size_t q = 0; q < shapes[g].size(); q++) map[q] = new_id[shapes[g][q]];
        DeviceScope scope(p.device);
        SPMVB_TRY(spmvb_pattern_remap(p.a, (int32_t)order.size(), offs.data(), flat.data(), ends.data(), map.data(), p.st));
    }
    return SPMVB_OK;
}

}  // namespace

extern "C" {

int spmvb_multi_create(const spmvb_grid *grid, int32_t format, const spmvb_compress_options *opts, const int32_t *devices,
                       int32_t n_devices, spmvb_multi **out) {
    if (!out) return fail(SPMVB_ERR_INVALID_ARGUMENT, "multi_create: out is NULL");
    *out = nullptr;
    if (!grid || !devices || n_devices < 1) return fail(SPMVB_ERR_INVALID_ARGUMENT, "multi_create: needs a grid and a device list");
    if (grid->nx < 1 || grid->ny < 1 || grid->nz < n_devices)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "multi_create: %d planes cannot be cut into %d slabs", grid->nz, n_devices);
    if (format != SPMVB_FMT_ELL && format != SPMVB_FMT_VT && format != SPMVB_FMT_PATTERN)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "multi_create: format %d has no SpMV kernel", format);
    int count = 0;
    SPMVB_CUDA(cudaGetDeviceCount(&count));
    for (int g = 0; g < n_devices; g++)
        if (devices[g] < 0 || devices[g] >= count) return fail(SPMVB_ERR_INVALID_ARGUMENT, "multi_create: no device %d", devices[g]);
    spmvb_compress_options o = opts ? *opts : spmvb_compress_options{256, 1, 1, 0};
    spmvb_multi *m = new spmvb_multi();
    m->grid = *grid;
    m->format = format;
    m->plane = (int64_t)grid->nx * grid->ny;
    m->parts.resize(n_devices);
    const int64_t base = grid->nz / n_devices, rem = grid->nz % n_devices;  // low slabs take the remainder (slab.py:SlabLayout)
    int rc = SPMVB_OK;
    for (int g = 0; g < n_devices && rc == SPMVB_OK; g++) {
        auto &p = m->parts[g];
        p.device = devices[g];
        p.z0 = g * base + std::min<int64_t>(g, rem);
        p.z1 = p.z0 + base + (g < rem ? 1 : 0);
        DeviceScope scope(p.device);
        for (int peer = 0; peer < n_devices; peer++)  // neighbours' planes are read in place by the ghost copies
            if (devices[peer] != p.device && (peer == g - 1 || peer == g + 1)) {
                int can = 0;
                if (cudaDeviceCanAccessPeer(&can, p.device, devices[peer]) == cudaSuccess && can) {
                    const cudaError_t e = cudaDeviceEnablePeerAccess(devices[peer], 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) rc = fail(SPMVB_ERR_CUDA, "peer access %d -> %d: %s", p.device, devices[peer], cudaGetErrorString(e));
                }
                (void)cudaGetLastError();
            }
        if (rc != SPMVB_OK) break;
        if (cudaStreamCreateWithFlags(&p.st, cudaStreamNonBlocking) != cudaSuccess || cudaEventCreate(&p.t0) != cudaSuccess ||
            cudaEventCreate(&p.t1) != cudaSuccess) {
            rc = fail(SPMVB_ERR_CUDA, "multi_create: stream / events on device %d: %s", p.device, cudaGetErrorString(cudaGetLastError()));
            break;
        }
        spmvb_matrix *csr = nullptr;
        rc = spmvb_generate_csr(grid, p.z0 * m->plane, p.z1 * m->plane, p.st, &csr);
        if (rc != SPMVB_OK) break;
        // slabs use the global ELL width (27 for grids of >= 3^3), so every slab streams the same bytes per row
        const int32_t width = std::min(grid->nx, 3) * std::min(grid->ny, 3) * std::min(grid->nz, 3);
        if (format == SPMVB_FMT_ELL) rc = spmvb_csr_to_ell(csr, width, p.st, &p.a);
        else if (format == SPMVB_FMT_VT) rc = spmvb_csr_compress_values(csr, &o, width, p.st, &p.a);
        else rc = spmvb_csr_compress_patterns(csr, &o, p.st, &p.a);
        spmvb_matrix_destroy(csr);
        if (rc != SPMVB_OK) break;
        const int64_t n = p.a->n;
        rc = spmvb_vec_alloc(n + 2 * m->plane, &p.x);
        if (rc == SPMVB_OK) rc = spmvb_vec_alloc(n, &p.y);
        if (rc == SPMVB_OK && cudaMemsetAsync(p.x, 0, (size_t)(n + 2 * m->plane) * 8, p.st) != cudaSuccess) rc = fail(SPMVB_ERR_CUDA, "memset failed");
        if (rc == SPMVB_OK) rc = spmvb_slab_create(p.a, m->plane, g > 0, g < n_devices - 1, &p.slab);
    }
    if (rc == SPMVB_OK && format == SPMVB_FMT_PATTERN && n_devices > 1) rc = merge_dictionaries(m);
    for (auto &p : m->parts)
        if (rc == SPMVB_OK && p.st) {
            DeviceScope scope(p.device);
            if (cudaStreamSynchronize(p.st) != cudaSuccess) rc = fail(SPMVB_ERR_CUDA, "multi_create: %s", cudaGetErrorString(cudaGetLastError()));
        }
    if (rc != SPMVB_OK) {
        const std::string keep = last_error_ref();
        multi_free(m);
        last_error_ref() = keep;
        return rc;
    }
    *out = m;
    return SPMVB_OK;
}

int spmvb_multi_destroy(spmvb_multi *m) {
    multi_free(m);
    return SPMVB_OK;
}

int spmvb_multi_parts(const spmvb_multi *m, int32_t *n_parts) {
    if (!m || !n_parts) return fail(SPMVB_ERR_INVALID_ARGUMENT, "NULL argument");
    *n_parts = (int32_t)m->parts.size();
    return SPMVB_OK;
}

int spmvb_multi_part(const spmvb_multi *m, int32_t part, int32_t *device, int64_t *z0, int64_t *z1, const spmvb_matrix **matrix,
                     double **x_ghosted, double **y) {
    if (!m || part < 0 || part >= (int)m->parts.size()) return fail(SPMVB_ERR_INVALID_ARGUMENT, "multi_part: no part %d", part);
    const auto &p = m->parts[part];
    if (device) *device = p.device;
    if (z0) *z0 = p.z0;
    if (z1) *z1 = p.z1;
    if (matrix) *matrix = p.a;
    if (x_ghosted) *x_ghosted = p.x;
    if (y) *y = p.y;
    return SPMVB_OK;
}

int spmvb_multi_sync(spmvb_multi *m) {
    if (!m) return fail(SPMVB_ERR_INVALID_ARGUMENT, "NULL argument");
    for (auto &p : m->parts) {
        DeviceScope scope(p.device);
        SPMVB_CUDA(cudaStreamSynchronize(p.st));
    }
    return SPMVB_OK;
}

int spmvb_multi_fill_x(spmvb_multi *m, int32_t kind, uint64_t seed, double lo, double hi) {
    if (!m) return fail(SPMVB_ERR_INVALID_ARGUMENT, "NULL argument");
    SPMVB_TRY(spmvb_multi_sync(m));  // nobody still reads the old x
    for (auto &p : m->parts) {  // owned entries only: element i is a pure function of (seed, global index); ghosts arrive by exchange
        DeviceScope scope(p.device);
        SPMVB_TRY(spmvb_vec_fill(p.x + m->plane, p.a->n, kind, seed, lo, hi, p.z0 * m->plane, p.st));
    }
    return spmvb_multi_sync(m);
}

int spmvb_multi_upload_x(spmvb_multi *m, const double *x_host, int64_t n) {
    if (!m || !x_host) return fail(SPMVB_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n != m->plane * m->grid.nz) return fail(SPMVB_ERR_INVALID_ARGUMENT, "multi: x has %lld entries, matrix has %lld rows", (long long)n, (long long)(m->plane * m->grid.nz));
    SPMVB_TRY(spmvb_multi_sync(m));
    for (auto &p : m->parts) {
        DeviceScope scope(p.device);
        SPMVB_CUDA(cudaMemcpyAsync(p.x + m->plane, x_host + p.z0 * m->plane, (size_t)p.a->n * 8, cudaMemcpyHostToDevice, p.st));
    }
    return spmvb_multi_sync(m);
}

int spmvb_multi_download_y(spmvb_multi *m, double *y_host, int64_t n) {
    if (!m || !y_host) return fail(SPMVB_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n != m->plane * m->grid.nz) return fail(SPMVB_ERR_INVALID_ARGUMENT, "multi: y has %lld entries, matrix has %lld rows", (long long)n, (long long)(m->plane * m->grid.nz));
    for (auto &p : m->parts) {
        DeviceScope scope(p.device);
        SPMVB_CUDA(cudaMemcpyAsync(y_host + p.z0 * m->plane, p.y, (size_t)p.a->n * 8, cudaMemcpyDeviceToHost, p.st));
    }
    return spmvb_multi_sync(m);
}

// One SpMV on every slab: each pulls its neighbours' boundary planes (x must be quiescent: the caller orders writes of x
// before this call, as spmvb_multi_fill_x / upload_x do) and runs its rows.  Asynchronous; one graph launch per slab.
int spmvb_multi_spmv(spmvb_multi *m, int32_t mode) {
    if (!m) return fail(SPMVB_ERR_INVALID_ARGUMENT, "NULL argument");
    const int G = (int)m->parts.size();
    for (int g = 0; g < G; g++) {
        auto &p = m->parts[g];
        const double *lo = g > 0 ? m->parts[g - 1].x + m->parts[g - 1].a->n : nullptr;  // the lower neighbour's last owned plane
        const double *hi = g < G - 1 ? m->parts[g + 1].x + m->plane : nullptr;          // the upper neighbour's first owned plane
        SPMVB_TRY(spmvb_slab_spmv(p.slab, p.x, p.y, lo, hi, mode, p.st));
    }
    return SPMVB_OK;
}

// reps SpMVs (exchange included) after one warm-up; host wall clock between device-wide syncs -> *seconds (all
// reps), and the slowest slab's device time between events -> *device_seconds (may be NULL).
int spmvb_multi_bench(spmvb_multi *m, int32_t reps, int32_t mode, double *seconds, double *device_seconds) {
    if (!m || reps < 1 || !seconds) return fail(SPMVB_ERR_INVALID_ARGUMENT, "multi_bench: bad arguments");
    for (int w = 0; w < 3; w++) SPMVB_TRY(spmvb_multi_spmv(m, mode));  // direct launches, graph capture, first replay
    SPMVB_TRY(spmvb_multi_sync(m));
    const auto t0 = std::chrono::steady_clock::now();
    for (auto &p : m->parts) {
        DeviceScope scope(p.device);
        SPMVB_CUDA(cudaEventRecord(p.t0, p.st));
    }
    for (int r = 0; r < reps; r++) SPMVB_TRY(spmvb_multi_spmv(m, mode));
    for (auto &p : m->parts) {
        DeviceScope scope(p.device);
        SPMVB_CUDA(cudaEventRecord(p.t1, p.st));
    }
    SPMVB_TRY(spmvb_multi_sync(m));
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (device_seconds) {
        float worst = 0.f;
        for (auto &p : m->parts) {
            DeviceScope scope(p.device);
            float ms = 0.f;
            SPMVB_CUDA(cudaEventElapsedTime(&ms, p.t0, p.t1));
            worst = std::max(worst, ms);
        }
        *device_seconds = worst * 1e-3;
    }
    return SPMVB_OK;
}

}  // extern "C"
