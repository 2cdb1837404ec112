// Device-side format builders: to_ell (inc/ell.hpp:28-29), compress_values
// (inc/compress.hpp:82), compress_patterns (inc/compress.hpp:84-85) with the
// exception-row extension, decompress / to_stencil (inc/compress.hpp:87-90,
// inc/ell.hpp:31-32) and validate (inc/compress.hpp:92-95).  All inputs and
// outputs are device-resident handles; only the small tables (value table,
// dictionary) pass through the host.
#include <cub/cub.cuh>

#include <algorithm>
#include <map>
#include <numeric>

#include "common.cuh"
#include "hash.cuh"

namespace spmvb {

int exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t count, cudaStream_t st);  // generate.cu

namespace {

struct DevBuf {  // RAII scratch
    void *p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
    int alloc(size_t bytes) {
        if (p) { cudaFree(p); p = nullptr; }
        cudaError_t e = cudaMalloc(&p, bytes ? bytes : 16);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            p = nullptr;
            return fail(SPMVB_ERR_NOMEM, "cudaMalloc of %zu scratch bytes failed: %s", bytes, cudaGetErrorString(e));
        }
        return SPMVB_OK;
    }
    template <class T> T *as() { return static_cast<T *>(p); }
};

struct Csr {
    const int64_t *row_start;
    const int32_t *cols;
    const double *vals;
    int n;
    int64_t row_offset;
};

Csr view(const spmvb_matrix *m) {
    return Csr{static_cast<const int64_t *>(m->s[SPMVB_S_CSR_ROW_START]), static_cast<const int32_t *>(m->s[SPMVB_S_CSR_COLS]),
               static_cast<const double *>(m->s[SPMVB_S_CSR_VALS]), m->n, m->row_offset};
}

int sync(cudaStream_t st, const char *what) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SPMVB_ERR_CUDA, "%s failed: %s", what, cudaGetErrorString(e));
    return SPMVB_OK;
}

int new_like(const spmvb_matrix *src, int format, spmvb_matrix **a) {
    *a = new spmvb_matrix();
    (*a)->device = src->device;
    (*a)->format = format;
    (*a)->n = src->n;
    (*a)->row_offset = src->row_offset;
    (*a)->n_cols = src->n_cols;
    return SPMVB_OK;
}

inline unsigned blocks_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

// ---- row-length reductions -----------------------------------------------------
__global__ void max_row_len_kernel(Csr m, int *out) {
    int best = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m.n; i += (int64_t)gridDim.x * blockDim.x)
        best = max(best, (int)(m.row_start[i + 1] - m.row_start[i]));
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best > 0) atomicMax(out, best);
}

int max_row_len(const Csr &m, cudaStream_t st, int *out) {
    DevBuf d;
    SPMVB_TRY(d.alloc(4));
    SPMVB_CUDA(cudaMemsetAsync(d.p, 0, 4, st));
    if (m.n > 0) max_row_len_kernel<<<std::min(blocks_for(m.n, 256), (unsigned)sm_count() * 8u), 256, 0, st>>>(m, d.as<int>());
    SPMVB_CUDA(cudaMemcpyAsync(out, d.p, 4, cudaMemcpyDeviceToHost, st));
    return sync(st, "max_row_len");
}

// ---- to_ell ------------------------------------------------------------------------
__global__ void to_ell_kernel(Csr m, int width, double *__restrict__ values, int32_t *__restrict__ columns) {
    // one warp per row: slots in ascending-column order, trailing padding (0.0, own row)
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= m.n) return;
    const int64_t b = m.row_start[row];
    const int k = (int)(m.row_start[row + 1] - b);
    const int64_t s = row * width;
    for (int t = lane; t < width; t += 32) {
        values[s + t] = t < k ? m.vals[b + t] : 0.0;
        columns[s + t] = t < k ? m.cols[b + t] : (int32_t)(m.row_offset + row);
    }
}

// ---- value table ---------------------------------------------------------------------
// Distinct values by bit pattern.  The table is tiny, the value stream
// is huge: each pass checks every value against the current table (binary search on
// the ascending table) and appends the misses to a bounded list; the host merges
// the list into the table and repeats until a pass has no miss.
constexpr int kMissCap = 1 << 16;

__device__ __forceinline__ bool dbl_less(double a, double b) {
    if (a < b) return true;
    if (a > b) return false;
    return (uint64_t)__double_as_longlong(a) < (uint64_t)__double_as_longlong(b);
}
__device__ __forceinline__ int table_find(const double *tab, int m, double v) {
    int lo = 0, hi = m;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (dbl_less(tab[mid], v)) lo = mid + 1; else hi = mid;
    }
    return (lo < m && __double_as_longlong(tab[lo]) == __double_as_longlong(v)) ? lo : -1;
}

__global__ void table_miss_kernel(const double *__restrict__ vals, int64_t nnz, const uint8_t *__restrict__ row_keep,
                                  const int64_t *__restrict__ row_start, int n, const double *__restrict__ tab, int m,
                                  double *__restrict__ miss, unsigned long long *__restrict__ n_miss) {
    // row_keep == nullptr: scan all values; otherwise only rows with row_keep[row] != 0
    if (row_keep == nullptr) {
        for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x) {
            const double v = vals[t];
            if (table_find(tab, m, v) < 0) {
                const unsigned long long slot = atomicAdd(n_miss, 1ULL);
                if (slot < kMissCap) miss[slot] = v;
            }
        }
    } else {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
            if (!row_keep[i]) continue;
            for (int64_t t = row_start[i]; t < row_start[i + 1]; t++) {
                const double v = vals[t];
                if (table_find(tab, m, v) < 0) {
                    const unsigned long long slot = atomicAdd(n_miss, 1ULL);
                    if (slot < kMissCap) miss[slot] = v;
                }
            }
        }
    }
}

bool host_dbl_less(double a, double b) {
    if (a < b) return true;
    if (a > b) return false;
    uint64_t ua, ub;
    memcpy(&ua, &a, 8);
    memcpy(&ub, &b, 8);
    return ua < ub;
}

// scan_value_table (inc/compress.hpp:80): ascending distinct values; TableOverflowError above `limit`.
int scan_value_table(const Csr &m, int64_t nnz, const uint8_t *row_keep, size_t limit, cudaStream_t st,
                     std::vector<double> *table) {
    table->clear();
    DevBuf d_tab, d_miss, d_cnt;
    SPMVB_TRY(d_tab.alloc((limit + 1) * 8));
    SPMVB_TRY(d_miss.alloc((size_t)kMissCap * 8));
    SPMVB_TRY(d_cnt.alloc(8));
    std::vector<double> miss(kMissCap);
    if (!row_keep && nnz > 0) {  // seed with the distinct values of a short prefix
        const size_t seed = (size_t)std::min<int64_t>(nnz, 4096);
        SPMVB_CUDA(cudaMemcpy(miss.data(), m.vals, seed * 8, cudaMemcpyDeviceToHost));
        table->assign(miss.begin(), miss.begin() + seed);
        std::sort(table->begin(), table->end(), host_dbl_less);
        table->erase(std::unique(table->begin(), table->end(), [](double a, double b) { return !memcmp(&a, &b, 8); }),
                     table->end());
        if (table->size() > limit) return fail(SPMVB_ERR_TABLE_OVERFLOW, "more than %zu distinct matrix values", limit);
    }
    for (int pass = 0; pass < 100000; pass++) {
        SPMVB_CUDA(cudaMemsetAsync(d_cnt.p, 0, 8, st));
        if (!table->empty())
            SPMVB_CUDA(cudaMemcpyAsync(d_tab.p, table->data(), table->size() * 8, cudaMemcpyHostToDevice, st));
        const int64_t work = row_keep ? m.n : nnz;
        if (work > 0)
            table_miss_kernel<<<std::min(blocks_for(work, 256), (unsigned)sm_count() * 16u), 256, 0, st>>>(
                m.vals, nnz, row_keep, m.row_start, m.n, d_tab.as<double>(), (int)table->size(), d_miss.as<double>(),
                d_cnt.as<unsigned long long>());
        unsigned long long n_miss = 0;
        SPMVB_CUDA(cudaMemcpyAsync(&n_miss, d_cnt.p, 8, cudaMemcpyDeviceToHost, st));
        SPMVB_TRY(sync(st, "value-table scan"));
        if (n_miss == 0) return SPMVB_OK;
        const size_t got = (size_t)std::min<unsigned long long>(n_miss, kMissCap);
        SPMVB_CUDA(cudaMemcpy(miss.data(), d_miss.p, got * 8, cudaMemcpyDeviceToHost));
        table->insert(table->end(), miss.begin(), miss.begin() + got);
        std::sort(table->begin(), table->end(), host_dbl_less);
        table->erase(std::unique(table->begin(), table->end(),
                                 [](double a, double b) { return !memcmp(&a, &b, 8); }),
                     table->end());
        if (table->size() > limit)
            return fail(SPMVB_ERR_TABLE_OVERFLOW, "more than %zu distinct matrix values", limit);
    }
    return fail(SPMVB_ERR_CUDA, "value-table scan did not converge");
}

// ---- compress_values ---------------------------------------------------------------------
// Per row: stable counting sort of the (ascending-column) entries by value index gives
// the (value ascending, column ascending) order of SPEC.md:142,177; ends are the
// exclusive prefix counts.
__global__ void vt_rows_kernel(Csr m, const double *__restrict__ tab, int mt, int width,
                               int32_t *__restrict__ sorted_columns, int32_t *__restrict__ ends,
                               int32_t *__restrict__ cursor) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= m.n) return;
    const int64_t b = m.row_start[row], e = m.row_start[row + 1];
    int32_t *en = ends + row * mt;
    int32_t *cu = cursor + row * mt;
    for (int k = 0; k < mt; k++) en[k] = 0;
    for (int64_t t = b; t < e; t++) en[table_find(tab, mt, m.vals[t])]++;
    int run = 0;
    for (int k = 0; k < mt; k++) { cu[k] = run; run += en[k]; en[k] = run; }
    int32_t *sc = sorted_columns + row * width;
    for (int64_t t = b; t < e; t++) sc[cu[table_find(tab, mt, m.vals[t])]++] = m.cols[t];
    for (int t = (int)(e - b); t < width; t++) sc[t] = (int32_t)(m.row_offset + row);  // padding, never read
}

// ---- compress_patterns ----------------------------------------------------------------------
// Row shape = (length, displacement[], value bits[]) in ascending-column order; two rows
// share a pattern iff their shapes are identical (inc/compress.hpp:48-51).  Shapes are
// hashed, rows sorted by hash (stable: ascending row inside a hash), and every row is then
// compared in full against the first row of its hash run, so the grouping is exact; a hash
// collision (unequal shapes in one run) restarts with another salt.
__device__ __forceinline__ uint64_t shape_hash(const Csr &m, int64_t row, uint64_t salt) {
    const int64_t b = m.row_start[row], e = m.row_start[row + 1];
    uint64_t h = sm64(salt ^ (uint64_t)(e - b));
    const int64_t g = m.row_offset + row;
    for (int64_t t = b; t < e; t++) {
        h = sm64(h ^ (uint64_t)(uint32_t)(int32_t)((int64_t)m.cols[t] - g));
        h = sm64(h ^ (uint64_t)__double_as_longlong(m.vals[t]));
    }
    return h;
}

__global__ void shape_hash_kernel(Csr m, uint64_t salt, uint64_t *__restrict__ keys, int32_t *__restrict__ rows) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= m.n) return;
    keys[row] = shape_hash(m, row, salt);
    rows[row] = (int32_t)row;
}

__global__ void run_heads_kernel(const uint64_t *__restrict__ keys, int n, int64_t *__restrict__ flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// seg[i] = (inclusive scan of flags) - 1; head_pos[seg] = i where flag set
__global__ void run_head_pos_kernel(const int64_t *__restrict__ excl, const uint64_t *__restrict__ keys, int n,
                                    int32_t *__restrict__ seg, int32_t *__restrict__ head_pos) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool head = (i == 0 || keys[i] != keys[i - 1]);
    const int32_t s = (int32_t)(excl[i] + (head ? 1 : 0) - 1);
    seg[i] = s;
    if (head) head_pos[s] = (int32_t)i;
}

__device__ bool same_shape(const Csr &m, int64_t r1, int64_t r2) {
    const int64_t b1 = m.row_start[r1], b2 = m.row_start[r2];
    const int64_t k = m.row_start[r1 + 1] - b1;
    if (k != m.row_start[r2 + 1] - b2) return false;
    const int64_t d = r2 - r1;
    for (int64_t t = 0; t < k; t++) {
        if ((int64_t)m.cols[b2 + t] - (int64_t)m.cols[b1 + t] != d) return false;
        if (__double_as_longlong(m.vals[b1 + t]) != __double_as_longlong(m.vals[b2 + t])) return false;
    }
    return true;
}

__global__ void verify_runs_kernel(Csr m, const int32_t *__restrict__ rows, const int32_t *__restrict__ seg,
                                   const int32_t *__restrict__ head_pos, int n, int *__restrict__ collision) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t rep = rows[head_pos[seg[i]]];
    if (rep != rows[i] && !same_shape(m, rep, rows[i])) *collision = 1;
}

__global__ void run_stats_kernel(const int32_t *__restrict__ rows, const int32_t *__restrict__ head_pos, int n_seg, int n,
                                 int32_t *__restrict__ first_row, int32_t *__restrict__ count) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    const int32_t b = head_pos[s];
    const int32_t e = (s + 1 < n_seg) ? head_pos[s + 1] : n;
    first_row[s] = rows[b];  // stable sort: smallest row of the run
    count[s] = e - b;
}

__global__ void assign_ids_kernel(const int32_t *__restrict__ rows, const int32_t *__restrict__ seg,
                                  const int32_t *__restrict__ seg_id, int n, int32_t *__restrict__ row_pattern,
                                  uint8_t *__restrict__ row_keep) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t id = seg_id[seg[i]];
    row_pattern[rows[i]] = id;
    if (row_keep) row_keep[rows[i]] = id >= 0;
}

__global__ void gather_rows_kernel(Csr m, const int32_t *__restrict__ which, int count, int maxlen,
                                   int32_t *__restrict__ len, int32_t *__restrict__ disp, double *__restrict__ vals) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= count) return;
    const int64_t row = which[q];
    const int64_t b = m.row_start[row];
    const int k = (int)(m.row_start[row + 1] - b);
    len[q] = k;
    for (int t = 0; t < k && t < maxlen; t++) {
        disp[q * maxlen + t] = (int32_t)((int64_t)m.cols[b + t] - (m.row_offset + row));
        vals[q * maxlen + t] = m.vals[b + t];
    }
}

__global__ void exc_flag_kernel(const int32_t *__restrict__ row_pattern, int n, int64_t *__restrict__ flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = row_pattern[i] < 0 ? 1 : 0;
}

__global__ void exc_list_kernel(Csr m, const int32_t *__restrict__ row_pattern, const int64_t *__restrict__ slot,
                                int32_t *__restrict__ exc_rows, int *__restrict__ w_exc) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m.n || row_pattern[i] >= 0) return;
    exc_rows[slot[i]] = (int32_t)i;
    atomicMax(w_exc, (int)(m.row_start[i + 1] - m.row_start[i]));
}

__global__ void exc_fill_kernel(Csr m, const int32_t *__restrict__ exc_rows, int n_exc, int w_exc,
                                double *__restrict__ values, int32_t *__restrict__ columns) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_exc) return;
    const int64_t row = exc_rows[q];
    const int64_t b = m.row_start[row];
    const int k = (int)(m.row_start[row + 1] - b);
    for (int t = 0; t < w_exc; t++) {
        values[q * w_exc + t] = t < k ? m.vals[b + t] : 0.0;
        columns[q * w_exc + t] = t < k ? m.cols[b + t] : (int32_t)(m.row_offset + row);
    }
}

// ---- to_csr (decompress) ------------------------------------------------------------------------
struct AnyFmt {
    int format, n, width, m, w_exc;
    int64_t row_offset;
    const double *values, *table, *exc_values;
    const int32_t *columns, *ends, *row_pattern, *disp_off, *disp, *ends_flat, *exc_columns, *exc_rows;
    const int64_t *exc_slot;  // per row: index into the exception block (exclusive scan of id<0)
};

__device__ int any_row(const AnyFmt &f, int64_t row, int32_t *cols, double *vals, bool write) {
    int k = 0;
    const int32_t own = (int32_t)(f.row_offset + row);
    if (f.format == SPMVB_FMT_ELL) {
        for (int t = 0; t < f.width; t++) {
            const double v = f.values[row * f.width + t];
            const int32_t c = f.columns[row * f.width + t];
            if (v == 0.0 && c == own) continue;  // padding slot (inc/ell.hpp:31-32)
            if (write) { cols[k] = c; vals[k] = v; }
            k++;
        }
    } else if (f.format == SPMVB_FMT_VT) {
        int idx = 0;
        for (int g = 0; g < f.m; g++)
            for (; idx < f.ends[row * f.m + g]; idx++) {
                if (write) { cols[k] = f.columns[row * f.width + idx]; vals[k] = f.table[g]; }
                k++;
            }
    } else {
        const int32_t id = f.row_pattern[row];
        if (id < 0) {
            const int64_t q = f.exc_slot[row];
            for (int t = 0; t < f.w_exc; t++) {
                const double v = f.exc_values[q * f.w_exc + t];
                const int32_t c = f.exc_columns[q * f.w_exc + t];
                if (v == 0.0 && c == own) continue;
                if (write) { cols[k] = c; vals[k] = v; }
                k++;
            }
        } else {
            const int32_t b = f.disp_off[id];
            int idx = 0;
            for (int g = 0; g < f.m; g++)
                for (; idx < f.ends_flat[id * f.m + g]; idx++) {
                    if (write) { cols[k] = own + f.disp[b + idx]; vals[k] = f.table[g]; }
                    k++;
                }
        }
    }
    return k;
}

__global__ void any_count_kernel(AnyFmt f, int64_t *__restrict__ counts) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row < f.n) counts[row] = any_row(f, row, nullptr, nullptr, false);
}

__global__ void any_fill_kernel(AnyFmt f, const int64_t *__restrict__ row_start, int32_t *__restrict__ cols,
                                double *__restrict__ vals) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= f.n) return;
    int32_t *c = cols + row_start[row];
    double *v = vals + row_start[row];
    const int k = any_row(f, row, c, v, true);
    for (int i = 1; i < k; i++) {  // columns re-sorted ascending (inc/compress.hpp:87-88)
        const int32_t ci = c[i];
        const double vi = v[i];
        int j = i - 1;
        while (j >= 0 && c[j] > ci) { c[j + 1] = c[j]; v[j + 1] = v[j]; j--; }
        c[j + 1] = ci;
        v[j + 1] = vi;
    }
}

// ---- validate ---------------------------------------------------------------------------------------
__global__ void validate_kernel(AnyFmt f, int n_patterns, int64_t n_cols, int *__restrict__ bad_row, int *__restrict__ bad_kind) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= f.n) return;
    int kind = 0;
    const int64_t own = f.row_offset + row;
    if (f.format == SPMVB_FMT_VT) {
        int prev = 0;
        for (int g = 0; g < f.m; g++) {
            const int e = f.ends[row * f.m + g];
            if (e < prev) kind = 1;  // non-monotone ends
            prev = e;
        }
        if (prev > f.width) kind = 1;
        for (int t = 0; t < prev && t < f.width && !kind; t++) {
            const int32_t c = f.columns[row * f.width + t];
            if (c < 0 || c >= n_cols) kind = 2;  // column out of range
        }
    } else if (f.format == SPMVB_FMT_PATTERN) {
        const int32_t id = f.row_pattern[row];
        if (id == -1) {
            const int64_t q = f.exc_slot[row];
            if (f.exc_rows[q] != row) kind = 4;  // exception list out of step with the ids
            for (int t = 0; t < f.w_exc && !kind; t++) {
                const int32_t c = f.exc_columns[q * f.w_exc + t];
                if (c < 0 || c >= n_cols) kind = 2;
            }
        } else if (id < 0 || id >= n_patterns) {
            kind = 3;  // pattern id out of range
        } else {
            for (int t = f.disp_off[id]; t < f.disp_off[id + 1]; t++) {
                const int64_t c = own + f.disp[t];
                if (c < 0 || c >= n_cols) kind = 2;
            }
        }
    } else if (f.format == SPMVB_FMT_ELL) {
        for (int t = 0; t < f.width; t++) {
            const int32_t c = f.columns[row * f.width + t];
            if (c < 0 || c >= n_cols) kind = 2;
        }
    }
    if (kind) {
        atomicMin(bad_row, (int)row);
        atomicMax(bad_kind, kind);
    }
}

__global__ void remap_ids_kernel(int32_t *__restrict__ row_pattern, int n, const int32_t *__restrict__ old_to_new, int n_old) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t id = row_pattern[i];
    if (id >= 0 && id < n_old) row_pattern[i] = old_to_new[id];
}

int build_any(const spmvb_matrix *a, DevBuf &slot_buf, cudaStream_t st, AnyFmt *f) {
    memset(f, 0, sizeof *f);
    f->format = a->format; f->n = a->n; f->width = a->width; f->m = a->m; f->w_exc = a->w_exc;
    f->row_offset = a->row_offset;
    if (a->format == SPMVB_FMT_ELL) {
        f->values = static_cast<const double *>(a->s[SPMVB_S_VALUES]);
        f->columns = static_cast<const int32_t *>(a->s[SPMVB_S_COLUMNS]);
    } else if (a->format == SPMVB_FMT_VT) {
        f->columns = static_cast<const int32_t *>(a->s[SPMVB_S_SORTED_COLUMNS]);
        f->ends = static_cast<const int32_t *>(a->s[SPMVB_S_ENDS]);
        f->table = static_cast<const double *>(a->s[SPMVB_S_TABLE]);
    } else if (a->format == SPMVB_FMT_PATTERN) {
        f->table = static_cast<const double *>(a->s[SPMVB_S_TABLE]);
        f->row_pattern = static_cast<const int32_t *>(a->s[SPMVB_S_ROW_PATTERN]);
        f->disp_off = a->d_disp_off32;
        f->disp = static_cast<const int32_t *>(a->s[SPMVB_S_DISP_FLAT]);
        f->ends_flat = static_cast<const int32_t *>(a->s[SPMVB_S_ENDS_FLAT]);
        f->exc_values = static_cast<const double *>(a->s[SPMVB_S_EXC_VALUES]);
        f->exc_columns = static_cast<const int32_t *>(a->s[SPMVB_S_EXC_COLUMNS]);
        f->exc_rows = static_cast<const int32_t *>(a->s[SPMVB_S_EXC_ROWS]);
        // per-row exception slot = exclusive scan of (id < 0)
        SPMVB_TRY(slot_buf.alloc((size_t)(a->n + 1) * 16));
        int64_t *flags = slot_buf.as<int64_t>();
        int64_t *slots = flags + a->n + 1;
        SPMVB_CUDA(cudaMemsetAsync(flags, 0, (size_t)(a->n + 1) * 8, st));
        if (a->n > 0) exc_flag_kernel<<<blocks_for(a->n, 256), 256, 0, st>>>(f->row_pattern, a->n, flags);
        SPMVB_TRY(exclusive_scan_i64(flags, slots, a->n + 1, st));
        f->exc_slot = slots;
    } else {
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "format %d cannot be decompressed", a->format);
    }
    return SPMVB_OK;
}

}  // namespace
}  // namespace spmvb

using namespace spmvb;

#define GUARD(call)               \
    do {                          \
        int rc__ = (call);        \
        if (rc__ != SPMVB_OK) {   \
            destroy(a);           \
            return rc__;          \
        }                         \
    } while (0)
#define GUARD_CUDA(expr)                                                                              \
    do {                                                                                              \
        cudaError_t e__ = (expr);                                                                     \
        if (e__ != cudaSuccess) {                                                                     \
            destroy(a);                                                                               \
            return fail(SPMVB_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e__));             \
        }                                                                                             \
    } while (0)

extern "C" {

int spmvb_csr_to_ell(const spmvb_matrix *csr, int32_t min_width, void *stream, spmvb_matrix **out) {
    if (!csr || !out || csr->format != SPMVB_FMT_CSR) return fail(SPMVB_ERR_INVALID_ARGUMENT, "csr_to_ell: needs a CSR handle");
    *out = nullptr;
    cudaStream_t st = as_stream(stream);
    const Csr m = view(csr);
    int width = 0;
    SPMVB_TRY(max_row_len(m, st, &width));
    width = std::max(width, (int)min_width);
    spmvb_matrix *a = nullptr;
    new_like(csr, SPMVB_FMT_ELL, &a);
    a->width = width;
    a->nnz = csr->nnz;
    const uint64_t slots = (uint64_t)csr->n * width;
    GUARD(dev_alloc(a, SPMVB_S_VALUES, slots * 8, (uint64_t)kTileRows * width * 8));
    GUARD(dev_alloc(a, SPMVB_S_COLUMNS, slots * 4, (uint64_t)kTileRows * width * 4));
    if (csr->n > 0 && width > 0)
        to_ell_kernel<<<blocks_for((int64_t)csr->n * 32, 256), 256, 0, st>>>(m, width, static_cast<double *>(a->s[SPMVB_S_VALUES]),
                                                                           static_cast<int32_t *>(a->s[SPMVB_S_COLUMNS]));
    GUARD(sync(st, "to_ell"));
    *out = a;
    return SPMVB_OK;
}

int spmvb_csr_compress_values(const spmvb_matrix *csr, const spmvb_compress_options *opts, int32_t min_width,
                              void *stream, spmvb_matrix **out) {
    if (!csr || !out || csr->format != SPMVB_FMT_CSR) return fail(SPMVB_ERR_INVALID_ARGUMENT, "compress_values: needs a CSR handle");
    *out = nullptr;
    cudaStream_t st = as_stream(stream);
    const Csr m = view(csr);
    const size_t limit = opts && opts->value_table_limit ? (size_t)opts->value_table_limit : 256;
    std::vector<double> table;
    SPMVB_TRY(scan_value_table(m, csr->nnz, nullptr, limit, st, &table));
    int width = 0;
    SPMVB_TRY(max_row_len(m, st, &width));
    width = std::max(width, (int)min_width);
    const int mt = (int)table.size();
    spmvb_matrix *a = nullptr;
    new_like(csr, SPMVB_FMT_VT, &a);
    a->width = width; a->m = mt; a->nnz = csr->nnz; a->h_table = table;
    GUARD(upload_stream(a, SPMVB_S_TABLE, table.data(), (uint64_t)mt * 8));
    GUARD(dev_alloc(a, SPMVB_S_SORTED_COLUMNS, (uint64_t)csr->n * width * 4, (uint64_t)kTileRows * width * 4));
    GUARD(dev_alloc(a, SPMVB_S_ENDS, (uint64_t)csr->n * mt * 4, (uint64_t)kTileRows * mt * 4));
    DevBuf cursor;
    GUARD(cursor.alloc((size_t)csr->n * std::max(mt, 1) * 4));
    if (csr->n > 0)
        vt_rows_kernel<<<blocks_for(csr->n, 128), 128, 0, st>>>(m, static_cast<const double *>(a->s[SPMVB_S_TABLE]), mt, width,
                                                              static_cast<int32_t *>(a->s[SPMVB_S_SORTED_COLUMNS]),
                                                              static_cast<int32_t *>(a->s[SPMVB_S_ENDS]), cursor.as<int32_t>());
    GUARD(sync(st, "compress_values"));
    *out = a;
    return SPMVB_OK;
}

int spmvb_csr_compress_patterns(const spmvb_matrix *csr, const spmvb_compress_options *opts, void *stream,
                                spmvb_matrix **out) {
    if (!csr || !out || csr->format != SPMVB_FMT_CSR) return fail(SPMVB_ERR_INVALID_ARGUMENT, "compress_patterns: needs a CSR handle");
    *out = nullptr;
    cudaStream_t st = as_stream(stream);
    const Csr m = view(csr);
    const int n = csr->n;
    const size_t limit = opts && opts->value_table_limit ? (size_t)opts->value_table_limit : 256;
    const int min_rows = opts && opts->min_pattern_rows > 1 ? opts->min_pattern_rows : 1;
    const int dict_cap = opts ? opts->dict_cap : 0;
    const int vip = opts ? opts->values_in_pattern : 0;

    // 1. exact grouping of the rows by shape
    DevBuf keys_a, keys_b, rows_a, rows_b, flags, excl, seg, head_pos, coll, sort_tmp;
    SPMVB_TRY(keys_a.alloc((size_t)n * 8)); SPMVB_TRY(keys_b.alloc((size_t)n * 8));
    SPMVB_TRY(rows_a.alloc((size_t)n * 4)); SPMVB_TRY(rows_b.alloc((size_t)n * 4));
    SPMVB_TRY(flags.alloc((size_t)(n + 1) * 8)); SPMVB_TRY(excl.alloc((size_t)(n + 1) * 8));
    SPMVB_TRY(seg.alloc((size_t)n * 4)); SPMVB_TRY(head_pos.alloc((size_t)(n + 1) * 4));
    SPMVB_TRY(coll.alloc(4));
    int n_seg = 0;
    const uint64_t *keys = nullptr;
    const int32_t *rows = nullptr;
    for (int attempt = 0;; attempt++) {
        if (attempt == 8) return fail(SPMVB_ERR_INTEGRITY, "compress_patterns: persistent hash collisions");
        if (n > 0) shape_hash_kernel<<<blocks_for(n, 128), 128, 0, st>>>(m, 0x5eed0000ULL + attempt, keys_a.as<uint64_t>(), rows_a.as<int32_t>());
        cub::DoubleBuffer<uint64_t> dk(keys_a.as<uint64_t>(), keys_b.as<uint64_t>());
        cub::DoubleBuffer<int32_t> dv(rows_a.as<int32_t>(), rows_b.as<int32_t>());
        size_t tmp_bytes = 0;
        SPMVB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, n, 0, 64, st));
        SPMVB_TRY(sort_tmp.alloc(tmp_bytes));
        SPMVB_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp.p, tmp_bytes, dk, dv, n, 0, 64, st));  // stable
        keys = dk.Current();
        rows = dv.Current();
        SPMVB_CUDA(cudaMemsetAsync(flags.p, 0, (size_t)(n + 1) * 8, st));
        if (n > 0) run_heads_kernel<<<blocks_for(n, 256), 256, 0, st>>>(keys, n, flags.as<int64_t>());
        SPMVB_TRY(exclusive_scan_i64(flags.as<int64_t>(), excl.as<int64_t>(), n + 1, st));
        int64_t total = 0;
        SPMVB_CUDA(cudaMemcpy(&total, excl.as<int64_t>() + n, 8, cudaMemcpyDeviceToHost));
        n_seg = (int)total;
        SPMVB_CUDA(cudaMemsetAsync(coll.p, 0, 4, st));
        if (n > 0) {
            run_head_pos_kernel<<<blocks_for(n, 256), 256, 0, st>>>(excl.as<int64_t>(), keys, n, seg.as<int32_t>(), head_pos.as<int32_t>());
            verify_runs_kernel<<<blocks_for(n, 128), 128, 0, st>>>(m, rows, seg.as<int32_t>(), head_pos.as<int32_t>(), n, coll.as<int>());
        }
        int collided = 0;
        SPMVB_CUDA(cudaMemcpyAsync(&collided, coll.p, 4, cudaMemcpyDeviceToHost, st));
        SPMVB_TRY(sync(st, "compress_patterns grouping"));
        if (!collided) break;
    }

    // 2. dictionary selection on the host: shapes used by >= min_rows rows; above dict_cap
    //    keep the most frequent (ties: earlier first row); ids by first occurrence in
    //    ascending row order (unpinned choice 1).
    DevBuf d_first, d_count, d_segid;
    SPMVB_TRY(d_first.alloc((size_t)std::max(n_seg, 1) * 4)); SPMVB_TRY(d_count.alloc((size_t)std::max(n_seg, 1) * 4));
    SPMVB_TRY(d_segid.alloc((size_t)std::max(n_seg, 1) * 4));
    if (n_seg > 0) run_stats_kernel<<<blocks_for(n_seg, 256), 256, 0, st>>>(rows, head_pos.as<int32_t>(), n_seg, n, d_first.as<int32_t>(), d_count.as<int32_t>());
    std::vector<int32_t> first(n_seg), count(n_seg), seg_id(n_seg, -1);
    SPMVB_CUDA(cudaMemcpyAsync(first.data(), d_first.p, (size_t)n_seg * 4, cudaMemcpyDeviceToHost, st));
    SPMVB_CUDA(cudaMemcpyAsync(count.data(), d_count.p, (size_t)n_seg * 4, cudaMemcpyDeviceToHost, st));
    SPMVB_TRY(sync(st, "compress_patterns stats"));
    std::vector<int32_t> kept;
    for (int s = 0; s < n_seg; s++)
        if (count[s] >= min_rows) kept.push_back(s);
    if (dict_cap > 0 && (int)kept.size() > dict_cap) {
        std::sort(kept.begin(), kept.end(), [&](int32_t x, int32_t y) {
            if (count[x] != count[y]) return count[x] > count[y];
            return first[x] < first[y];
        });
        kept.resize(dict_cap);
    }
    std::sort(kept.begin(), kept.end(), [&](int32_t x, int32_t y) { return first[x] < first[y]; });
    const int P = (int)kept.size();
    for (int p = 0; p < P; p++) seg_id[kept[p]] = p;

    // 3. representative rows of the kept shapes -> host -> table + dictionary
    int maxlen = 0;
    SPMVB_TRY(max_row_len(m, st, &maxlen));
    std::vector<int32_t> rep(P);
    for (int p = 0; p < P; p++) rep[p] = first[kept[p]];
    DevBuf d_rep, d_len, d_disp, d_vals;
    SPMVB_TRY(d_rep.alloc((size_t)std::max(P, 1) * 4)); SPMVB_TRY(d_len.alloc((size_t)std::max(P, 1) * 4));
    SPMVB_TRY(d_disp.alloc((size_t)std::max(P, 1) * std::max(maxlen, 1) * 4));
    SPMVB_TRY(d_vals.alloc((size_t)std::max(P, 1) * std::max(maxlen, 1) * 8));
    std::vector<int32_t> len(P), disp((size_t)P * maxlen);
    std::vector<double> vals((size_t)P * maxlen);
    if (P > 0) {
        SPMVB_CUDA(cudaMemcpyAsync(d_rep.p, rep.data(), (size_t)P * 4, cudaMemcpyHostToDevice, st));
        gather_rows_kernel<<<blocks_for(P, 128), 128, 0, st>>>(m, d_rep.as<int32_t>(), P, maxlen, d_len.as<int32_t>(), d_disp.as<int32_t>(), d_vals.as<double>());
        SPMVB_CUDA(cudaMemcpyAsync(len.data(), d_len.p, (size_t)P * 4, cudaMemcpyDeviceToHost, st));
        SPMVB_CUDA(cudaMemcpyAsync(disp.data(), d_disp.p, disp.size() * 4, cudaMemcpyDeviceToHost, st));
        SPMVB_CUDA(cudaMemcpyAsync(vals.data(), d_vals.p, vals.size() * 8, cudaMemcpyDeviceToHost, st));
        SPMVB_TRY(sync(st, "compress_patterns gather"));
    }
    // value table over dictionary rows only (exception rows keep their raw values)
    std::vector<double> table;
    for (int p = 0; p < P; p++)
        for (int t = 0; t < len[p]; t++) table.push_back(vals[(size_t)p * maxlen + t]);
    std::sort(table.begin(), table.end(), host_dbl_less);
    table.erase(std::unique(table.begin(), table.end(), [](double x, double y) { return !memcmp(&x, &y, 8); }), table.end());
    if (table.size() > limit) return fail(SPMVB_ERR_TABLE_OVERFLOW, "more than %zu distinct matrix values", limit);
    const int mt = (int)table.size();
    auto vidx = [&](double v) {
        return (int)(std::lower_bound(table.begin(), table.end(), v, host_dbl_less) - table.begin());
    };
    std::vector<int64_t> disp_offsets(P + 1, 0);
    std::vector<int32_t> disp_flat, ends_flat((size_t)P * mt, 0);
    for (int p = 0; p < P; p++) {
        std::vector<std::pair<int, int32_t>> e;  // (value index, displacement): sort = (value asc, disp asc)
        for (int t = 0; t < len[p]; t++) e.emplace_back(vidx(vals[(size_t)p * maxlen + t]), disp[(size_t)p * maxlen + t]);
        std::sort(e.begin(), e.end());
        size_t idx = 0;
        for (int g = 0; g < mt; g++) {
            while (idx < e.size() && e[idx].first == g) idx++;
            ends_flat[(size_t)p * mt + g] = (int32_t)idx;
        }
        for (auto &kv : e) disp_flat.push_back(kv.second);
        disp_offsets[p + 1] = (int64_t)disp_flat.size();
    }

    // 4. the handle: ids, dictionary, exception block
    spmvb_matrix *a = nullptr;
    new_like(csr, SPMVB_FMT_PATTERN, &a);
    a->m = mt; a->n_patterns = P; a->values_in_pattern = vip; a->nnz = csr->nnz;
    a->disp_total = (int64_t)disp_flat.size();
    a->h_table = table; a->h_disp_offsets = disp_offsets; a->h_disp_flat = disp_flat; a->h_ends_flat = ends_flat;
    a->h_first_rows = rep;
    GUARD(upload_stream(a, SPMVB_S_TABLE, table.data(), (uint64_t)mt * 8));
    GUARD(upload_stream(a, SPMVB_S_DISP_OFFSETS, disp_offsets.data(), (uint64_t)(P + 1) * 8));
    GUARD(upload_stream(a, SPMVB_S_DISP_FLAT, disp_flat.data(), (uint64_t)disp_flat.size() * 4));
    GUARD(upload_stream(a, SPMVB_S_ENDS_FLAT, ends_flat.data(), (uint64_t)ends_flat.size() * 4));
    GUARD(dev_alloc(a, SPMVB_S_ROW_PATTERN, (uint64_t)n * 4, 4096));
    GUARD_CUDA(cudaMemcpyAsync(d_segid.p, seg_id.data(), (size_t)n_seg * 4, cudaMemcpyHostToDevice, st));
    if (n > 0)
        assign_ids_kernel<<<blocks_for(n, 256), 256, 0, st>>>(rows, seg.as<int32_t>(), d_segid.as<int32_t>(), n,
                                                            static_cast<int32_t *>(a->s[SPMVB_S_ROW_PATTERN]), nullptr);
    // exception rows: ascending list, width = max exception row length, ELL block
    int32_t *row_pattern = static_cast<int32_t *>(a->s[SPMVB_S_ROW_PATTERN]);
    GUARD_CUDA(cudaMemsetAsync(flags.p, 0, (size_t)(n + 1) * 8, st));
    if (n > 0) exc_flag_kernel<<<blocks_for(n, 256), 256, 0, st>>>(row_pattern, n, flags.as<int64_t>());
    GUARD(exclusive_scan_i64(flags.as<int64_t>(), excl.as<int64_t>(), n + 1, st));
    int64_t n_exc64 = 0;
    GUARD_CUDA(cudaMemcpy(&n_exc64, excl.as<int64_t>() + n, 8, cudaMemcpyDeviceToHost));
    const int n_exc = (int)n_exc64;
    a->n_exc = n_exc;
    GUARD(dev_alloc(a, SPMVB_S_EXC_ROWS, (uint64_t)n_exc * 4, (uint64_t)kTileRows * 4));
    int w_exc = 0;
    if (n_exc > 0) {
        GUARD_CUDA(cudaMemsetAsync(coll.p, 0, 4, st));
        exc_list_kernel<<<blocks_for(n, 256), 256, 0, st>>>(m, row_pattern, excl.as<int64_t>(), static_cast<int32_t *>(a->s[SPMVB_S_EXC_ROWS]), coll.as<int>());
        GUARD_CUDA(cudaMemcpyAsync(&w_exc, coll.p, 4, cudaMemcpyDeviceToHost, st));
        GUARD(sync(st, "compress_patterns exceptions"));
    }
    a->w_exc = w_exc;
    GUARD(dev_alloc(a, SPMVB_S_EXC_VALUES, (uint64_t)n_exc * w_exc * 8, (uint64_t)kTileRows * w_exc * 8));
    GUARD(dev_alloc(a, SPMVB_S_EXC_COLUMNS, (uint64_t)n_exc * w_exc * 4, (uint64_t)kTileRows * w_exc * 4));
    if (n_exc > 0) {
        exc_fill_kernel<<<blocks_for(n_exc, 128), 128, 0, st>>>(m, static_cast<const int32_t *>(a->s[SPMVB_S_EXC_ROWS]), n_exc, w_exc,
                                                              static_cast<double *>(a->s[SPMVB_S_EXC_VALUES]),
                                                              static_cast<int32_t *>(a->s[SPMVB_S_EXC_COLUMNS]));
        a->h_exc_rows.resize(n_exc);
        GUARD_CUDA(cudaMemcpyAsync(a->h_exc_rows.data(), a->s[SPMVB_S_EXC_ROWS], (size_t)n_exc * 4, cudaMemcpyDeviceToHost, st));
    }
    GUARD(sync(st, "compress_patterns"));
    GUARD(finish_pattern_handle(a));
    *out = a;
    return SPMVB_OK;
}

int spmvb_to_csr(const spmvb_matrix *src, void *stream, spmvb_matrix **out) {
    if (!src || !out) return fail(SPMVB_ERR_INVALID_ARGUMENT, "to_csr: NULL argument");
    *out = nullptr;
    cudaStream_t st = as_stream(stream);
    if (src->format != SPMVB_FMT_ELL) SPMVB_TRY(spmvb_validate(src, INT64_MAX, stream));  // decompress validates first
    DevBuf slot_buf, counts;
    AnyFmt f;
    SPMVB_TRY(build_any(src, slot_buf, st, &f));
    const int n = src->n;
    SPMVB_TRY(counts.alloc((size_t)(n + 1) * 8));
    SPMVB_CUDA(cudaMemsetAsync(counts.p, 0, (size_t)(n + 1) * 8, st));
    if (n > 0) any_count_kernel<<<blocks_for(n, 128), 128, 0, st>>>(f, counts.as<int64_t>());
    spmvb_matrix *a = nullptr;
    new_like(src, SPMVB_FMT_CSR, &a);
    GUARD(dev_alloc(a, SPMVB_S_CSR_ROW_START, (uint64_t)(n + 1) * 8));
    GUARD(exclusive_scan_i64(counts.as<int64_t>(), static_cast<int64_t *>(a->s[SPMVB_S_CSR_ROW_START]), n + 1, st));
    int64_t nnz = 0;
    GUARD_CUDA(cudaMemcpy(&nnz, static_cast<int64_t *>(a->s[SPMVB_S_CSR_ROW_START]) + n, 8, cudaMemcpyDeviceToHost));
    a->nnz = nnz;
    GUARD(dev_alloc(a, SPMVB_S_CSR_COLS, (uint64_t)nnz * 4));
    GUARD(dev_alloc(a, SPMVB_S_CSR_VALS, (uint64_t)nnz * 8));
    if (n > 0)
        any_fill_kernel<<<blocks_for(n, 128), 128, 0, st>>>(f, static_cast<const int64_t *>(a->s[SPMVB_S_CSR_ROW_START]),
                                                          static_cast<int32_t *>(a->s[SPMVB_S_CSR_COLS]),
                                                          static_cast<double *>(a->s[SPMVB_S_CSR_VALS]));
    GUARD(sync(st, "to_csr"));
    *out = a;
    return SPMVB_OK;
}

int spmvb_validate(const spmvb_matrix *a, int64_t n_cols, void *stream) {
    if (!a) return fail(SPMVB_ERR_INVALID_ARGUMENT, "validate: NULL argument");
    cudaStream_t st = as_stream(stream);
    if (a->format == SPMVB_FMT_CSR) return SPMVB_OK;  // validated at construction (inc/stencil.hpp:47-48)
    for (size_t k = 1; k < a->h_table.size(); k++)
        if (!(a->h_table[k - 1] < a->h_table[k])) return fail(SPMVB_ERR_INTEGRITY, "value table not strictly ascending at %zu", k);
    if (a->format == SPMVB_FMT_PATTERN) {
        for (int p = 0; p < a->n_patterns; p++) {
            int32_t prev = 0;
            for (int k = 0; k < a->m; k++) {
                const int32_t e = a->h_ends_flat[(size_t)p * a->m + k];
                if (e < prev) return fail(SPMVB_ERR_INTEGRITY, "pattern %d: ends not monotone", p);
                prev = e;
            }
            if (prev != a->h_disp_offsets[p + 1] - a->h_disp_offsets[p])
                return fail(SPMVB_ERR_INTEGRITY, "pattern %d: last end %d != displacement count", p, prev);
        }
    }
    DevBuf slot_buf, bad;
    AnyFmt f;
    SPMVB_TRY(build_any(a, slot_buf, st, &f));
    if (a->format == SPMVB_FMT_PATTERN) {  // the exception list must match the ids == -1, in order
        int64_t n_exc = 0;
        SPMVB_CUDA(cudaMemcpy(&n_exc, f.exc_slot + a->n, 8, cudaMemcpyDeviceToHost));
        if (n_exc != a->n_exc) return fail(SPMVB_ERR_INTEGRITY, "exception list has %d rows, ids mark %lld", a->n_exc, (long long)n_exc);
    }
    SPMVB_TRY(bad.alloc(8));
    const int init[2] = {INT32_MAX, 0};
    SPMVB_CUDA(cudaMemcpyAsync(bad.p, init, 8, cudaMemcpyHostToDevice, st));
    if (a->n > 0) validate_kernel<<<blocks_for(a->n, 128), 128, 0, st>>>(f, a->n_patterns, n_cols, bad.as<int>(), bad.as<int>() + 1);
    int res[2] = {0, 0};
    SPMVB_CUDA(cudaMemcpyAsync(res, bad.p, 8, cudaMemcpyDeviceToHost, st));
    SPMVB_TRY(sync(st, "validate"));
    if (res[1]) {
        static const char *kinds[] = {"", "ends not monotone", "column out of range", "pattern id out of range",
                                      "exception list out of step with the pattern ids"};
        return fail(SPMVB_ERR_INTEGRITY, "row %d: %s", res[0], kinds[res[1]]);
    }
    return SPMVB_OK;
}

int spmvb_pattern_remap(spmvb_matrix *a, int32_t n_patterns, const int64_t *disp_offsets, const int32_t *disp_flat,
                        const int32_t *ends_flat, const int32_t *old_to_new, void *stream) {
    if (!a || a->format != SPMVB_FMT_PATTERN || !disp_offsets || !old_to_new)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "pattern_remap: needs a pattern handle");
    cudaStream_t st = as_stream(stream);
    const int n_old = a->n_patterns;
    DevBuf map;
    SPMVB_TRY(map.alloc((size_t)std::max(n_old, 1) * 4));
    SPMVB_CUDA(cudaMemcpyAsync(map.p, old_to_new, (size_t)n_old * 4, cudaMemcpyHostToDevice, st));
    if (a->n > 0)
        remap_ids_kernel<<<blocks_for(a->n, 256), 256, 0, st>>>(static_cast<int32_t *>(a->s[SPMVB_S_ROW_PATTERN]), a->n, map.as<int32_t>(), n_old);
    SPMVB_TRY(sync(st, "pattern_remap"));
    for (int sid : {SPMVB_S_DISP_OFFSETS, SPMVB_S_DISP_FLAT, SPMVB_S_ENDS_FLAT}) {
        if (a->s[sid]) cudaFree(a->s[sid]);
        a->s[sid] = nullptr;
        a->bytes[sid] = 0;
    }
    a->n_patterns = n_patterns;
    a->h_first_rows.clear();
    a->disp_total = disp_offsets[n_patterns];
    a->h_disp_offsets.assign(disp_offsets, disp_offsets + n_patterns + 1);
    a->h_disp_flat.assign(disp_flat, disp_flat + a->disp_total);
    a->h_ends_flat.assign(ends_flat, ends_flat + (size_t)n_patterns * a->m);
    SPMVB_TRY(upload_stream(a, SPMVB_S_DISP_OFFSETS, disp_offsets, (uint64_t)(n_patterns + 1) * 8));
    SPMVB_TRY(upload_stream(a, SPMVB_S_DISP_FLAT, disp_flat, (uint64_t)a->disp_total * 4));
    SPMVB_TRY(upload_stream(a, SPMVB_S_ENDS_FLAT, ends_flat, (uint64_t)n_patterns * a->m * 4));
    return finish_pattern_handle(a);
}

}  // extern "C"
