// C-ABI core: handles, upload / download, vectors, options.
// The declarations (with the reference file:line each replaces) are in
// include/spmvcomp_b200.h.
#include <algorithm>
#include <cmath>
#include <map>

#include "common.cuh"

namespace spmvb {

std::string &last_error_ref() {
    static thread_local std::string e;
    return e;
}

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    last_error_ref() = buf;
    return code;
}

Options &options() {  // per host thread: distinct handles driven by distinct threads do not see each other's knobs
    static thread_local Options o;
    return o;
}

int dev_alloc(spmvb_matrix *a, int sid, uint64_t bytes, uint64_t slack) {
    void *p = nullptr;
    uint64_t total = bytes + slack + 16;
    cudaError_t e = cudaMalloc(&p, total);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? SPMVB_ERR_NOMEM : SPMVB_ERR_CUDA,
                    "cudaMalloc of %llu bytes failed: %s", (unsigned long long)total, cudaGetErrorString(e));
    }
    SPMVB_CUDA(cudaMemset(static_cast<char *>(p) + bytes, 0, slack + 16));
    a->s[sid] = p;
    a->bytes[sid] = bytes;
    return SPMVB_OK;
}

int upload_stream(spmvb_matrix *a, int sid, const void *host, uint64_t bytes, uint64_t slack) {
    SPMVB_TRY(dev_alloc(a, sid, bytes, slack));
    if (bytes) SPMVB_CUDA(cudaMemcpy(a->s[sid], host, bytes, cudaMemcpyHostToDevice));
    return SPMVB_OK;
}

void destroy(spmvb_matrix *a) {
    if (!a) return;
    for (int i = 0; i < SPMVB_S_COUNT_; i++)
        if (a->s[i]) cudaFree(a->s[i]);
    if (a->scratch_x) cudaFree(a->scratch_x);
    if (a->scratch_y) cudaFree(a->scratch_y);
    if (a->cg_ws) cudaFree(a->cg_ws);
    if (a->symgs_graph.exec) cudaGraphExecDestroy(a->symgs_graph.exec);
    if (a->symgs_graph.capture_stream) cudaStreamDestroy(a->symgs_graph.capture_stream);
    for (auto &st : a->pipe_streams) if (st) cudaStreamDestroy(st);
    for (auto &ev : a->pipe_events) if (ev) cudaEventDestroy(ev);
    for (auto &ev : a->pipe_out_events) if (ev) cudaEventDestroy(ev);
    if (a->exc_stream) cudaStreamDestroy(a->exc_stream);
    for (auto &ev : a->exc_events) if (ev) cudaEventDestroy(ev);
    if (a->d_masks) cudaFree(a->d_masks);
    if (a->d_disp_off32) cudaFree(a->d_disp_off32);
    if (a->symgs_mask) cudaFree(a->symgs_mask);
    delete a;
}

// Looks for the sliding-window structure in the dictionary (see BoxPlan).
// Everything is derived from the reference's dictionary as uploaded; the
// dictionary layout itself is not changed.
void analyse_box_plan(spmvb_matrix *a) {
    BoxPlan &bp = a->box;
    bp = BoxPlan();
    const int P = a->n_patterns, m = a->m;
    if (P < 1 || m < 1 || m > 2) return;
    // candidate: a pattern with exactly 27 displacements
    for (int p = 0; p < P && !bp.valid; p++) {
        const int64_t b = a->h_disp_offsets[p], e = a->h_disp_offsets[p + 1];
        if (e - b != 27) continue;
        // (displacement -> value index) of this pattern
        std::map<int32_t, int32_t> dv;
        int idx = 0;
        for (int k = 0; k < m; k++)
            for (; idx < a->h_ends_flat[(size_t)p * m + k]; idx++) dv[a->h_disp_flat[b + idx]] = k;
        if (dv.size() != 27) continue;
        std::vector<int32_t> d;
        for (auto &kv : dv) d.push_back(kv.first);  // ascending
        if (d[13] != 0) continue;
        const int64_t sy = (int64_t)d[16] - d[13], sz = (int64_t)d[22] - d[13];
        if (sy <= 2 || sz <= 2 + 2 * sy || sz % sy != 0) continue;
        bool ok = true;
        for (int t = 0; t < 27 && ok; t++) {
            const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
            ok = d[t] == dx + sy * dy + sz * dz;
        }
        if (!ok) continue;
        const int kc = dv[0];
        int ko = -1;
        for (auto &kv : dv) {
            if (kv.first == 0) continue;
            if (ko < 0) ko = kv.second;
            if (kv.second != ko) ok = false;
        }
        if (!ok) continue;
        bp.valid = true;
        bp.sy = (int32_t)sy;
        bp.sz = (int32_t)sz;
        bp.k_off = ko;
        bp.k_center = kc;
        bp.center_pos = ko < kc ? 1 : (ko > kc ? 0 : 2);
    }
    if (!bp.valid) return;
    // every pattern: a sub-box with the same value per displacement -> 27-bit mask
    bp.masks.assign(P, kGenericMask);
    for (int p = 0; p < P; p++) {
        const int64_t b = a->h_disp_offsets[p];
        uint32_t mask = 0;
        bool ok = true;
        int idx = 0;
        for (int k = 0; k < m && ok; k++)
            for (; idx < a->h_ends_flat[(size_t)p * m + k] && ok; idx++) {
                const int64_t d = a->h_disp_flat[b + idx];
                // decode d = dx + sy*dy + sz*dz with dx,dy,dz in {-1,0,1}
                int found = -1;
                for (int t = 0; t < 27; t++) {
                    const int dx = t % 3 - 1, dy = (t / 3) % 3 - 1, dz = t / 9 - 1;
                    if (d == dx + (int64_t)bp.sy * dy + (int64_t)bp.sz * dz) { found = t; break; }
                }
                if (found < 0 || (mask >> found & 1u)) { ok = false; break; }
                const int want = found == 13 ? bp.k_center : bp.k_off;
                if (k != want) { ok = false; break; }
                mask |= 1u << found;
            }
        if (ok) bp.masks[p] = mask;
    }
}

// Smallest and largest global column referenced by the rows of a pattern handle (ids + per-pattern displacement
// extremes, plus the exception block).  out[0] = min, out[1] = max.
__global__ void column_range_kernel(const int32_t *__restrict__ ids, int n, int64_t row_offset, const int32_t *__restrict__ pmin,
                                    const int32_t *__restrict__ pmax, int n_patterns, const int32_t *__restrict__ exc_cols,
                                    int64_t n_exc_entries, long long *out) {
    long long lo = INT64_MAX, hi = INT64_MIN;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t r = t0; r < n; r += stride) {
        const int id = ids[r];
        if (id >= 0 && id < n_patterns) {  // (a malformed id is reported by validate; never an out-of-bounds read here)
            lo = min(lo, (long long)(row_offset + r + pmin[id]));
            hi = max(hi, (long long)(row_offset + r + pmax[id]));
        }
    }
    for (int64_t e = t0; e < n_exc_entries; e += stride) {
        lo = min(lo, (long long)exc_cols[e]);
        hi = max(hi, (long long)exc_cols[e]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (lo != INT64_MAX) atomicMin(out, lo);
        if (hi != INT64_MIN) atomicMax(out + 1, hi);
    }
}

static int compute_column_range(spmvb_matrix *a) {
    a->col_min = 0;
    a->col_max = -1;
    const int P = a->n_patterns;
    if (a->n <= 0 || P <= 0 || !a->s[SPMVB_S_ROW_PATTERN]) return SPMVB_OK;
    std::vector<int32_t> ext(2 * (size_t)P);
    for (int p = 0; p < P; p++) {
        int32_t lo = 0, hi = 0;
        const int64_t b = a->h_disp_offsets[p], e = a->h_disp_offsets[p + 1];
        if (e > b) {
            lo = hi = a->h_disp_flat[b];
            for (int64_t t = b; t < e; t++) lo = std::min(lo, a->h_disp_flat[t]), hi = std::max(hi, a->h_disp_flat[t]);
        }
        ext[p] = lo;
        ext[P + p] = hi;
    }
    int32_t *d_ext = nullptr;
    long long *d_out = nullptr;
    SPMVB_CUDA(cudaMalloc(&d_ext, ext.size() * sizeof(int32_t)));
    SPMVB_CUDA(cudaMalloc(&d_out, 2 * sizeof(long long)));
    const long long init[2] = {INT64_MAX, INT64_MIN};
    long long res[2];
    cudaError_t e1 = cudaMemcpy(d_ext, ext.data(), ext.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    cudaError_t e2 = cudaMemcpy(d_out, init, sizeof(init), cudaMemcpyHostToDevice);
    if (e1 == cudaSuccess && e2 == cudaSuccess) {
        column_range_kernel<<<592, 256>>>(static_cast<const int32_t *>(a->s[SPMVB_S_ROW_PATTERN]), a->n, a->row_offset, d_ext, d_ext + P, P,
                                          static_cast<const int32_t *>(a->s[SPMVB_S_EXC_COLUMNS]), (int64_t)a->n_exc * a->w_exc, d_out);
        e1 = cudaGetLastError();
        e2 = cudaMemcpy(res, d_out, sizeof(res), cudaMemcpyDeviceToHost);
    }
    cudaFree(d_ext);
    cudaFree(d_out);
    if (e1 != cudaSuccess || e2 != cudaSuccess)
        return fail(SPMVB_ERR_CUDA, "column range scan failed: %s", cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    if (res[0] <= res[1]) a->col_min = res[0], a->col_max = res[1];
    return SPMVB_OK;
}

int finish_pattern_handle(spmvb_matrix *a) {
    analyse_box_plan(a);
    SPMVB_TRY(compute_column_range(a));
    const int P = a->n_patterns;
    std::vector<uint32_t> masks = a->box.masks;
    if (masks.empty()) masks.assign(std::max(P, 1), kGenericMask);
    if (a->d_masks) { cudaFree(a->d_masks); a->d_masks = nullptr; }
    if (a->d_disp_off32) { cudaFree(a->d_disp_off32); a->d_disp_off32 = nullptr; }
    SPMVB_CUDA(cudaMalloc(&a->d_masks, masks.size() * sizeof(uint32_t)));
    SPMVB_CUDA(cudaMemcpy(a->d_masks, masks.data(), masks.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    std::vector<int32_t> off32(P + 1);
    for (int p = 0; p <= P; p++) off32[p] = (int32_t)a->h_disp_offsets[p];
    SPMVB_CUDA(cudaMalloc(&a->d_disp_off32, off32.size() * sizeof(int32_t)));
    SPMVB_CUDA(cudaMemcpy(a->d_disp_off32, off32.data(), off32.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    return SPMVB_OK;
}

}  // namespace spmvb

using namespace spmvb;

extern "C" {

const char *spmvb_last_error(void) { return last_error_ref().c_str(); }

int spmvb_version(void) { return 100; }

int spmvb_device_count(int *count) {
    if (!count) return fail(SPMVB_ERR_INVALID_ARGUMENT, "count is NULL");
    *count = 0;
    SPMVB_CUDA(cudaGetDeviceCount(count));
    return SPMVB_OK;
}

int spmvb_set_device(int device) {
    SPMVB_CUDA(cudaSetDevice(device));
    return SPMVB_OK;
}

static int *option_slot(const char *key) {
    if (!key) return nullptr;
    Options &o = options();
    if (!strcmp(key, "pattern_kernel")) return &o.pattern_kernel;
    if (!strcmp(key, "ell_kernel")) return &o.ell_kernel;
    if (!strcmp(key, "box_march")) return &o.box_march;
    if (!strcmp(key, "box_prefetch")) return &o.box_prefetch;
    if (!strcmp(key, "box_prefetch_l1")) return &o.box_prefetch_l1;
    if (!strcmp(key, "debug_nochain")) return &o.debug_nochain;
    if (!strcmp(key, "box_lines")) return &o.box_lines;
    if (!strcmp(key, "ring_leftover")) return &o.ring_leftover;
    if (!strcmp(key, "ring_pdl")) return &o.ring_pdl;
    if (!strcmp(key, "ring_two_lines")) return &o.ring_two_lines;
    if (!strcmp(key, "ring_min_steps")) return &o.ring_min_steps;
    if (!strcmp(key, "exception_kernel")) return &o.exception_kernel;
    if (!strcmp(key, "exception_overlap")) return &o.exception_overlap;
    if (!strcmp(key, "exception_carveout")) return &o.exception_carveout;
    if (!strcmp(key, "host_chunks")) return &o.host_chunks;
    if (!strcmp(key, "host_stage")) return &o.host_stage;
    if (!strcmp(key, "host_copy_threads")) return &o.host_copy_threads;
    if (!strcmp(key, "cg_keep_workspace")) return &o.cg_keep_workspace;
    if (!strcmp(key, "cg_fused_dot")) return &o.cg_fused_dot;
    if (!strcmp(key, "cg_graph")) return &o.cg_graph;
    if (!strcmp(key, "cg_pdl")) return &o.cg_pdl;
    if (!strcmp(key, "cg_fused_scalars")) return &o.cg_fused_scalars;
    if (!strcmp(key, "last_cg_graph")) return &o.last_cg_graph;
    if (!strcmp(key, "last_symgs_kernel")) return &o.last_symgs_kernel;
    if (!strcmp(key, "symgs_graph")) return &o.symgs_graph;
    if (!strcmp(key, "symgs_persistent")) return &o.symgs_persistent;
    if (!strcmp(key, "symgs_pipeline")) return &o.symgs_pipeline;
    if (!strcmp(key, "symgs_lag")) return &o.symgs_lag;
    if (!strcmp(key, "slab_graph")) return &o.slab_graph;
    if (!strcmp(key, "last_cg_fused_dot")) return &o.last_cg_fused_dot;
    if (!strcmp(key, "last_pattern_kernel")) return &o.last_pattern_kernel;
    return nullptr;
}

// Values that select measured experiments / ablations exist only in the lab build (-DSPMVB_LAB); the default library
// rejects them, so no option can make it return a wrong y.
static bool lab_only_value(const char *key, int value) {
    if (kLabBuild) return false;
    if (!strcmp(key, "box_march")) {
        for (int ok : {0, 3, 90, 101, 107, 108, 109, 110, 111, 112})
            if (value == ok) return false;
        return true;
    }
    if (!strcmp(key, "debug_nochain")) return value != 0;
    if (!strcmp(key, "ell_kernel")) return value < 0 || value > 3;
    if (!strcmp(key, "pattern_kernel")) return value < 0 || value > 3;
    return false;
}

int spmvb_set_option(const char *key, int value) {
    int *s = option_slot(key);
    if (!s) return fail(SPMVB_ERR_INVALID_ARGUMENT, "unknown option '%s'", key ? key : "(null)");
    if (lab_only_value(key, value))
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "option '%s' = %d selects a lab variant; this library was built without -DSPMVB_LAB", key, value);
    *s = value;
    return SPMVB_OK;
}

int spmvb_get_option(const char *key, int *value) {
    if (key && value && !strcmp(key, "lab_build")) {
        *value = kLabBuild ? 1 : 0;
        return SPMVB_OK;
    }
    int *s = option_slot(key);
    if (!s || !value) return fail(SPMVB_ERR_INVALID_ARGUMENT, "unknown option '%s'", key ? key : "(null)");
    *value = *s;
    return SPMVB_OK;
}

static int new_handle(spmvb_matrix **out, spmvb_matrix **a) {
    if (!out) return fail(SPMVB_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    int dev = 0;
    SPMVB_CUDA(cudaGetDevice(&dev));
    *a = new spmvb_matrix();
    (*a)->device = dev;
    return SPMVB_OK;
}

#define GUARD(call)               \
    do {                          \
        int rc__ = (call);        \
        if (rc__ != SPMVB_OK) {   \
            destroy(a);           \
            return rc__;          \
        }                         \
    } while (0)

int spmvb_ell_upload(int32_t n, int32_t width, int64_t nnz, int64_t row_offset, const double *values,
                     const int32_t *columns, spmvb_matrix **out) {
    if (n < 0 || width < 0 || (n > 0 && width > 0 && (!values || !columns)))
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "ell_upload: bad arguments (n=%d width=%d)", n, width);
    spmvb_matrix *a = nullptr;
    SPMVB_TRY(new_handle(out, &a));
    a->format = SPMVB_FMT_ELL;
    a->n = n; a->width = width; a->nnz = nnz; a->row_offset = row_offset;
    const uint64_t slots = (uint64_t)n * (uint64_t)width;
    const uint64_t slack_rows = kTileRows;
    GUARD(upload_stream(a, SPMVB_S_VALUES, values, slots * 8, slack_rows * width * 8));
    GUARD(upload_stream(a, SPMVB_S_COLUMNS, columns, slots * 4, slack_rows * width * 4));
    *out = a;
    return SPMVB_OK;
}

int spmvb_vt_upload(int32_t n, int32_t width, int32_t m, int64_t row_offset, const double *table,
                    const int32_t *sorted_columns, const int32_t *ends, spmvb_matrix **out) {
    if (n < 0 || width < 0 || m < 0 || (n > 0 && (!sorted_columns || !ends || !table)))
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "vt_upload: bad arguments");
    spmvb_matrix *a = nullptr;
    SPMVB_TRY(new_handle(out, &a));
    a->format = SPMVB_FMT_VT;
    a->n = n; a->width = width; a->m = m; a->row_offset = row_offset;
    a->h_table.assign(table, table + m);
    int64_t nnz = 0;
    for (int64_t i = 0; i < n && m > 0; i++) nnz += ends[(i + 1) * (int64_t)m - 1];
    a->nnz = nnz;
    GUARD(upload_stream(a, SPMVB_S_TABLE, table, (uint64_t)m * 8));
    GUARD(upload_stream(a, SPMVB_S_SORTED_COLUMNS, sorted_columns, (uint64_t)n * width * 4,
                        (uint64_t)kTileRows * width * 4));
    GUARD(upload_stream(a, SPMVB_S_ENDS, ends, (uint64_t)n * m * 4, (uint64_t)kTileRows * m * 4));
    *out = a;
    return SPMVB_OK;
}

int spmvb_pattern_upload(int32_t n, int32_t m, int64_t row_offset, const double *table,
                         int32_t n_patterns, const int64_t *disp_offsets, const int32_t *disp_flat,
                         const int32_t *ends_flat, const int32_t *row_pattern, int32_t values_in_pattern,
                         int32_t n_exc, int32_t w_exc, const int32_t *exc_rows, const double *exc_values,
                         const int32_t *exc_columns, spmvb_matrix **out) {
    if (n < 0 || m < 0 || n_patterns < 0 || n_exc < 0 || w_exc < 0 || !disp_offsets || (m > 0 && !table) ||
        (n_patterns > 0 && m > 0 && !ends_flat) || (n > 0 && !row_pattern) ||
        (n_exc > 0 && (!exc_rows || (w_exc > 0 && (!exc_values || !exc_columns)))))
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "pattern_upload: bad arguments");
    // structural checks on the small tables (validate(), inc/compress.hpp:92-95)
    for (int k = 1; k < m; k++)
        if (!(table[k - 1] < table[k]))
            return fail(SPMVB_ERR_INTEGRITY, "value table not strictly ascending at %d", k);
    if (disp_offsets[0] != 0) return fail(SPMVB_ERR_INTEGRITY, "disp_offsets[0] != 0");
    for (int p = 0; p < n_patterns; p++) {
        const int64_t len = disp_offsets[p + 1] - disp_offsets[p];
        int32_t prev = 0;
        for (int k = 0; k < m; k++) {
            const int32_t e = ends_flat[(size_t)p * m + k];
            if (e < prev) return fail(SPMVB_ERR_INTEGRITY, "pattern %d: ends not monotone", p);
            prev = e;
        }
        if (len < 0 || prev != len)
            return fail(SPMVB_ERR_INTEGRITY, "pattern %d: last end %d != displacement count %lld", p, prev,
                        (long long)len);
    }
    if (disp_offsets[n_patterns] > INT32_MAX)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "dictionary too large");
    if (disp_offsets[n_patterns] > 0 && !disp_flat) return fail(SPMVB_ERR_INVALID_ARGUMENT, "pattern_upload: disp_flat is NULL");
    // the row stream and the exception list, before anything reaches the device: ids in [-1, P), the exception rows
    // ascending, in range, and exactly the rows whose id is -1
    int64_t nnz = 0, n_minus1 = 0;
    for (int64_t i = 0; i < n; i++) {
        const int32_t id = row_pattern[i];
        if (id >= 0 && id < n_patterns) nnz += disp_offsets[id + 1] - disp_offsets[id];
        else if (id == -1) n_minus1++;
        else return fail(SPMVB_ERR_INTEGRITY, "row %lld: pattern id %d out of range", (long long)i, id);
    }
    if (n_minus1 != n_exc) return fail(SPMVB_ERR_INTEGRITY, "%lld rows have id -1 but the exception block holds %d rows", (long long)n_minus1, n_exc);
    for (int64_t e = 0; e < n_exc; e++) {
        const int32_t r = exc_rows[e];
        if (r < 0 || r >= n || (e > 0 && r <= exc_rows[e - 1]) || row_pattern[r] != -1)
            return fail(SPMVB_ERR_INTEGRITY, "exception slot %lld: row %d is out of range, out of order or has a pattern id", (long long)e, r);
        for (int32_t t = 0; t < w_exc; t++)
            if (!(exc_values[e * w_exc + t] == 0.0 && exc_columns[e * w_exc + t] == row_offset + r)) nnz++;
    }
    spmvb_matrix *a = nullptr;
    SPMVB_TRY(new_handle(out, &a));
    a->format = SPMVB_FMT_PATTERN;
    a->n = n; a->m = m; a->row_offset = row_offset; a->n_patterns = n_patterns;
    a->values_in_pattern = values_in_pattern; a->n_exc = n_exc; a->w_exc = w_exc;
    a->disp_total = disp_offsets[n_patterns];
    a->h_table.assign(table, table + m);
    a->h_disp_offsets.assign(disp_offsets, disp_offsets + n_patterns + 1);
    a->h_disp_flat.assign(disp_flat, disp_flat + a->disp_total);
    a->h_ends_flat.assign(ends_flat, ends_flat + (size_t)n_patterns * m);
    if (n_exc) a->h_exc_rows.assign(exc_rows, exc_rows + n_exc);
    GUARD(upload_stream(a, SPMVB_S_TABLE, table, (uint64_t)m * 8));
    GUARD(upload_stream(a, SPMVB_S_DISP_OFFSETS, disp_offsets, (uint64_t)(n_patterns + 1) * 8));
    GUARD(upload_stream(a, SPMVB_S_DISP_FLAT, disp_flat, (uint64_t)a->disp_total * 4));
    GUARD(upload_stream(a, SPMVB_S_ENDS_FLAT, ends_flat, (uint64_t)n_patterns * m * 4));
    GUARD(upload_stream(a, SPMVB_S_ROW_PATTERN, row_pattern, (uint64_t)n * 4, 4096));
    GUARD(upload_stream(a, SPMVB_S_EXC_ROWS, exc_rows, (uint64_t)n_exc * 4, (uint64_t)kTileRows * 4));
    GUARD(upload_stream(a, SPMVB_S_EXC_VALUES, exc_values, (uint64_t)n_exc * w_exc * 8,
                        (uint64_t)kTileRows * w_exc * 8));
    GUARD(upload_stream(a, SPMVB_S_EXC_COLUMNS, exc_columns, (uint64_t)n_exc * w_exc * 4,
                        (uint64_t)kTileRows * w_exc * 4));
    GUARD(finish_pattern_handle(a));
    a->nnz = nnz;  // pattern rows via the dictionary, exception rows via non-padding slots
    *out = a;
    return SPMVB_OK;
}

int spmvb_csr_upload(int32_t n, int64_t n_cols, int64_t row_offset, const int64_t *row_start,
                     const int32_t *cols, const double *vals, spmvb_matrix **out) {
    if (n < 0 || !row_start || row_start[0] != 0)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "csr_upload: bad arguments");
    for (int64_t i = 0; i < n; i++) {  // stencil_from_rows contract, inc/stencil.hpp:47-48
        if (row_start[i + 1] < row_start[i]) return fail(SPMVB_ERR_INVALID_ARGUMENT, "row_start not monotone at %lld", (long long)i);
        for (int64_t t = row_start[i]; t < row_start[i + 1]; t++) {
            if (cols[t] < 0 || cols[t] >= n_cols)
                return fail(SPMVB_ERR_INVALID_ARGUMENT, "row %lld: column %d out of range", (long long)i, cols[t]);
            if (t > row_start[i] && cols[t] <= cols[t - 1])
                return fail(SPMVB_ERR_INVALID_ARGUMENT, "row %lld: columns not strictly ascending", (long long)i);
        }
    }
    spmvb_matrix *a = nullptr;
    SPMVB_TRY(new_handle(out, &a));
    a->format = SPMVB_FMT_CSR;
    a->n = n; a->n_cols = n_cols; a->row_offset = row_offset; a->nnz = row_start[n];
    GUARD(upload_stream(a, SPMVB_S_CSR_ROW_START, row_start, (uint64_t)(n + 1) * 8));
    GUARD(upload_stream(a, SPMVB_S_CSR_COLS, cols, (uint64_t)a->nnz * 4));
    GUARD(upload_stream(a, SPMVB_S_CSR_VALS, vals, (uint64_t)a->nnz * 8));
    *out = a;
    return SPMVB_OK;
}

int spmvb_matrix_get_info(const spmvb_matrix *a, spmvb_matrix_info *info) {
    if (!a || !info) return fail(SPMVB_ERR_INVALID_ARGUMENT, "NULL argument");
    memset(info, 0, sizeof *info);
    info->format = a->format; info->n = a->n; info->width = a->width; info->m = a->m;
    info->n_patterns = a->n_patterns; info->n_exc = a->n_exc; info->w_exc = a->w_exc;
    info->values_in_pattern = a->values_in_pattern; info->nnz = a->nnz; info->row_offset = a->row_offset;
    info->disp_total = a->disp_total; info->device = a->device;
    info->kernel_plan = a->box.valid ? 1 : 0;
    info->box_stride_y = a->box.sy; info->box_stride_z = a->box.sz;
    return SPMVB_OK;
}

int spmvb_matrix_stream_bytes(const spmvb_matrix *a, int32_t sid, uint64_t *bytes) {
    if (!a || !bytes || sid < 0 || sid >= SPMVB_S_COUNT_) return fail(SPMVB_ERR_INVALID_ARGUMENT, "bad stream id %d", sid);
    *bytes = a->s[sid] ? a->bytes[sid] : 0;
    return SPMVB_OK;
}

int spmvb_matrix_download(const spmvb_matrix *a, int32_t sid, uint64_t offset, uint64_t bytes, void *dst) {
    if (!a || sid < 0 || sid >= SPMVB_S_COUNT_) return fail(SPMVB_ERR_INVALID_ARGUMENT, "bad stream id %d", sid);
    if (!a->s[sid] || offset + bytes > a->bytes[sid])
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "stream %d: range [%llu,+%llu) outside %llu bytes", sid,
                    (unsigned long long)offset, (unsigned long long)bytes, (unsigned long long)a->bytes[sid]);
    if (bytes) SPMVB_CUDA(cudaMemcpy(dst, static_cast<const char *>(a->s[sid]) + offset, bytes, cudaMemcpyDeviceToHost));
    return SPMVB_OK;
}

int spmvb_matrix_stream_ptr(const spmvb_matrix *a, int32_t sid, void **dev_ptr) {
    if (!a || !dev_ptr || sid < 0 || sid >= SPMVB_S_COUNT_) return fail(SPMVB_ERR_INVALID_ARGUMENT, "bad stream id %d", sid);
    *dev_ptr = a->s[sid];
    return SPMVB_OK;
}

int spmvb_pattern_first_rows(const spmvb_matrix *a, int32_t *out) {
    if (!a || !out || a->format != SPMVB_FMT_PATTERN) return fail(SPMVB_ERR_INVALID_ARGUMENT, "first_rows: needs a pattern handle");
    for (int p = 0; p < a->n_patterns; p++) out[p] = p < (int)a->h_first_rows.size() ? a->h_first_rows[p] : -1;
    return SPMVB_OK;
}

int spmvb_matrix_destroy(spmvb_matrix *a) {
    destroy(a);
    return SPMVB_OK;
}

// ---- vectors -------------------------------------------------------------------
int spmvb_vec_alloc(int64_t n, double **dev) {
    if (n < 0 || !dev) return fail(SPMVB_ERR_INVALID_ARGUMENT, "vec_alloc: bad arguments");
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, (size_t)(n > 0 ? n : 1) * 8);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? SPMVB_ERR_NOMEM : SPMVB_ERR_CUDA, "cudaMalloc failed: %s",
                    cudaGetErrorString(e));
    }
    *dev = static_cast<double *>(p);
    return SPMVB_OK;
}

int spmvb_vec_free(double *dev) {
    if (dev) SPMVB_CUDA(cudaFree(dev));
    return SPMVB_OK;
}

int spmvb_vec_upload(double *dev, const double *host, int64_t n, void *stream) {
    SPMVB_CUDA(cudaMemcpyAsync(dev, host, (size_t)n * 8, cudaMemcpyHostToDevice, as_stream(stream)));
    SPMVB_CUDA(cudaStreamSynchronize(as_stream(stream)));
    return SPMVB_OK;
}

int spmvb_vec_download(double *host, const double *dev, int64_t n, void *stream) {
    SPMVB_CUDA(cudaMemcpyAsync(host, dev, (size_t)n * 8, cudaMemcpyDeviceToHost, as_stream(stream)));
    SPMVB_CUDA(cudaStreamSynchronize(as_stream(stream)));
    return SPMVB_OK;
}

}  // extern "C"
