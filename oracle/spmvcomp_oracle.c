/*
 * spmvcomp_oracle.c -- CPU ORACLE (TEST INFRASTRUCTURE, NOT PRODUCT CODE).
 * See spmvcomp_oracle.h for scope, pins and the "parity unpinned" list.
 * Reference citations are file:line under /root/reference
 * (inc/ = proj/include/spmvcomp/).
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared -pthread (oracle/Makefile).
 */
#include "spmvcomp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
const char *orc_last_error(void) { return g_err; }
#define FAIL(code, ...)                                \
    do {                                               \
        snprintf(g_err, sizeof g_err, __VA_ARGS__);    \
        return (code);                                 \
    } while (0)

/* ------------------------------------------------------------------------- */
/* counter-based hashing (UNPINNED choice (2)/(4): splitmix64 finaliser)      */
/* ------------------------------------------------------------------------- */
static inline uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t h2(uint64_t seed, uint64_t a) { return sm64(sm64(seed) ^ a); }
static inline uint64_t h3(uint64_t seed, uint64_t a, uint64_t b) {
    return sm64(h2(seed, a) ^ (b * 0xD6E8FEB86659FD93ULL));
}
static inline double u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

/* ------------------------------------------------------------------------- */
/* generator                                                                  */
/* ------------------------------------------------------------------------- */
#define ORC_MAX_ROW 32 /* 27 stencil entries + up to 4 added */

/* One row of the 27-point stencil (inc/stencil.hpp:40-45): node
 * (ix,iy,iz) couples to every in-grid (ix+dx,iy+dy,iz+dz); out-of-grid
 * couplings are omitted; row id = ix + nx*(iy + ny*iz)
 * (inc/grid.hpp:13-14).  dz,dy,dx ascending enumerates columns ascending. */
static int stencil_row(int nx, int ny, int nz, double diag, double off, int64_t row,
                       int32_t *cols, double *vals) {
    int ix = (int)(row % nx);
    int iy = (int)((row / nx) % ny);
    int iz = (int)(row / ((int64_t)nx * ny));
    int k = 0;
    for (int dz = -1; dz <= 1; dz++) {
        int z = iz + dz;
        if (z < 0 || z >= nz) continue;
        for (int dy = -1; dy <= 1; dy++) {
            int y = iy + dy;
            if (y < 0 || y >= ny) continue;
            for (int dx = -1; dx <= 1; dx++) {
                int x = ix + dx;
                if (x < 0 || x >= nx) continue;
                int64_t c = x + (int64_t)nx * (y + (int64_t)ny * z);
                cols[k] = (int32_t)c;
                vals[k] = (c == row) ? diag : off;
                k++;
            }
        }
    }
    return k;
}

/* Config-4 perturbation (BASELINE.json configs[3]; recipe fixed in DESIGN.md
 * "C4 recipe", UNPINNED choice (4)).  Pure function of (seed, row). */
static int perturb_row(const orc_perturb *p, int64_t n, int64_t row, int32_t *cols, double *vals,
                       int k, double diag, double off) {
    if (!(u01(h3(p->seed, (uint64_t)row, 0)) < p->fraction)) return k;
    int steps = 1 + (int)(h3(p->seed, (uint64_t)row, 1) & 3);
    for (int s = 0; s < steps; s++) {
        uint64_t hs = h3(p->seed, (uint64_t)row, 2 + (uint64_t)s);
        int n_off = k - 1;
        int drop = ((hs & 1) == 0) && n_off > 0;
        if (drop) {
            int j = (int)((hs >> 1) % (uint64_t)n_off); /* j-th off-diagonal, ascending */
            int pos = -1, seen = 0;
            for (int t = 0; t < k; t++) {
                if (cols[t] == row) continue;
                if (seen == j) { pos = t; break; }
                seen++;
            }
            for (int t = pos; t + 1 < k; t++) { cols[t] = cols[t + 1]; vals[t] = vals[t + 1]; }
            k--;
        } else {
            if ((int64_t)k >= n) continue; /* row already full */
            int64_t c = (int64_t)((hs >> 1) % (uint64_t)n);
            for (;;) { /* linear probe to the next absent column */
                int present = 0;
                for (int t = 0; t < k; t++) if (cols[t] == c) { present = 1; break; }
                if (!present) break;
                c = (c + 1) % n;
            }
            int pos = k;
            while (pos > 0 && cols[pos - 1] > c) { cols[pos] = cols[pos - 1]; vals[pos] = vals[pos - 1]; pos--; }
            cols[pos] = (int32_t)c;
            vals[pos] = off;
            k++;
        }
    }
    /* off-diagonals: off + (2u-1)*noise, one rounding per operation; diagonal :=
     * sum |off-diagonal| in ascending column order (keeps weak dominance). */
    double sum = 0.0;
    int t_off = 0, dpos = -1;
    for (int t = 0; t < k; t++) {
        if (cols[t] == row) { dpos = t; continue; }
        double u = u01(h3(p->seed, (uint64_t)row, 16 + (uint64_t)t_off));
        double w = (2.0 * u - 1.0) * p->noise;
        vals[t] = off + w;
        sum = sum + fabs(vals[t]);
        t_off++;
    }
    if (dpos >= 0) vals[dpos] = (t_off > 0) ? sum : diag;
    return k;
}

typedef struct rowgen {
    int nx, ny, nz;
    double diag, off;
    orc_perturb pert;
    int64_t n;
    const orc_csr *csr; /* when non-NULL rows come from here */
} rowgen;

static int rowgen_row(const rowgen *g, int64_t row, int32_t *cols, double *vals) {
    if (g->csr) {
        int64_t b = g->csr->row_start[row], e = g->csr->row_start[row + 1];
        memcpy(cols, g->csr->cols + b, (size_t)(e - b) * sizeof(int32_t));
        memcpy(vals, g->csr->vals + b, (size_t)(e - b) * sizeof(double));
        return (int)(e - b);
    }
    int k = stencil_row(g->nx, g->ny, g->nz, g->diag, g->off, row, cols, vals);
    if (g->pert.enabled) k = perturb_row(&g->pert, g->n, row, cols, vals, k, g->diag, g->off);
    return k;
}

static int check_grid(int nx, int ny, int nz) {
    /* inc/grid.hpp:35-47 */
    if (nx < 1 || ny < 1 || nz < 1)
        FAIL(ORC_INVALID_ARGUMENT, "grid dimensions must be >= 1, got %dx%dx%d", nx, ny, nz);
    if ((int64_t)nx * ny * nz > (((int64_t)1 << 31) - 1) || (double)nx * ny * nz > 2147483647.0)
        FAIL(ORC_INVALID_ARGUMENT, "grid %dx%dx%d: column indices must fit a 4-byte signed integer", nx, ny, nz);
    return ORC_OK;
}

int orc_generate_rows(int nx, int ny, int nz, double diagonal, double off_diagonal,
                      const orc_perturb *p, int64_t row_begin, int64_t row_end, orc_csr **out) {
    int rc = check_grid(nx, ny, nz);
    if (rc) return rc;
    int64_t n = (int64_t)nx * ny * nz;
    if (row_begin < 0 || row_end > n || row_begin > row_end)
        FAIL(ORC_INVALID_ARGUMENT, "row range [%lld,%lld) outside [0,%lld)", (long long)row_begin,
             (long long)row_end, (long long)n);
    rowgen g = {nx, ny, nz, diagonal, off_diagonal, {0, 0, 0, 0}, n, NULL};
    if (p && p->enabled) g.pert = *p;
    int64_t nl = row_end - row_begin;
    orc_csr *m = calloc(1, sizeof *m);
    if (!m) FAIL(ORC_NOMEM, "out of memory");
    m->n = (int32_t)nl;
    m->nx = nx; m->ny = ny; m->nz = nz;
    size_t cap = (size_t)nl * (g.pert.enabled ? 28 : 27) + 64;
    m->row_start = malloc((size_t)(nl + 1) * sizeof(int64_t));
    m->cols = malloc(cap * sizeof(int32_t));
    m->vals = malloc(cap * sizeof(double));
    if (!m->row_start || !m->cols || !m->vals) { orc_csr_free(m); FAIL(ORC_NOMEM, "out of memory"); }
    int64_t pos = 0;
    int32_t c[ORC_MAX_ROW];
    double v[ORC_MAX_ROW];
    for (int64_t r = 0; r < nl; r++) {
        m->row_start[r] = pos;
        int k = rowgen_row(&g, row_begin + r, c, v);
        if ((size_t)(pos + k) > cap) {
            cap = cap + cap / 4 + 64;
            m->cols = realloc(m->cols, cap * sizeof(int32_t));
            m->vals = realloc(m->vals, cap * sizeof(double));
            if (!m->cols || !m->vals) { orc_csr_free(m); FAIL(ORC_NOMEM, "out of memory"); }
        }
        memcpy(m->cols + pos, c, (size_t)k * sizeof(int32_t));
        memcpy(m->vals + pos, v, (size_t)k * sizeof(double));
        pos += k;
    }
    m->row_start[nl] = pos;
    *out = m;
    return ORC_OK;
}

int orc_csr_from_arrays(int32_t n, const int64_t *row_start, const int32_t *cols,
                        const double *vals, orc_csr **out) {
    /* inc/stencil.hpp:47-50: columns strictly ascending and in [0,n) */
    if (n < 0 || row_start[0] != 0) FAIL(ORC_INVALID_ARGUMENT, "bad row_start");
    for (int32_t i = 0; i < n; i++) {
        if (row_start[i + 1] < row_start[i]) FAIL(ORC_INVALID_ARGUMENT, "row_start not monotone at %d", i);
        for (int64_t t = row_start[i]; t < row_start[i + 1]; t++) {
            if (cols[t] < 0 || cols[t] >= n) FAIL(ORC_INVALID_ARGUMENT, "row %d: column %d out of range", i, cols[t]);
            if (t > row_start[i] && cols[t] <= cols[t - 1]) FAIL(ORC_INVALID_ARGUMENT, "row %d: columns not strictly ascending", i);
        }
    }
    orc_csr *m = calloc(1, sizeof *m);
    int64_t nnz = row_start[n];
    m->n = n;
    m->row_start = malloc((size_t)(n + 1) * sizeof(int64_t));
    m->cols = malloc((size_t)(nnz + 1) * sizeof(int32_t));
    m->vals = malloc((size_t)(nnz + 1) * sizeof(double));
    memcpy(m->row_start, row_start, (size_t)(n + 1) * sizeof(int64_t));
    memcpy(m->cols, cols, (size_t)nnz * sizeof(int32_t));
    memcpy(m->vals, vals, (size_t)nnz * sizeof(double));
    *out = m;
    return ORC_OK;
}

void orc_csr_free(orc_csr *m) {
    if (!m) return;
    free(m->row_start); free(m->cols); free(m->vals); free(m);
}

int orc_csr_equal(const orc_csr *a, const orc_csr *b) {
    /* inc/stencil.hpp:24,38: grid provenance excluded from equality */
    if (a->n != b->n) return 0;
    if (memcmp(a->row_start, b->row_start, (size_t)(a->n + 1) * sizeof(int64_t))) return 0;
    int64_t nnz = a->row_start[a->n];
    return !memcmp(a->cols, b->cols, (size_t)nnz * sizeof(int32_t)) &&
           !memcmp(a->vals, b->vals, (size_t)nnz * sizeof(double));
}

static int64_t csr_find(const orc_csr *m, int32_t i, int32_t j) {
    int64_t lo = m->row_start[i], hi = m->row_start[i + 1];
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (m->cols[mid] < j) lo = mid + 1; else hi = mid;
    }
    return (lo < m->row_start[i + 1] && m->cols[lo] == j) ? lo : -1;
}

int orc_is_symmetric(const orc_csr *m) {
    /* (i,j,v) present <=> (j,i,v) present */
    for (int32_t i = 0; i < m->n; i++)
        for (int64_t t = m->row_start[i]; t < m->row_start[i + 1]; t++) {
            int64_t u = csr_find(m, m->cols[t], i);
            if (u < 0 || memcmp(&m->vals[u], &m->vals[t], sizeof(double))) return 0;
        }
    return 1;
}

int orc_make_test_vector(int64_t n, int kind, uint64_t seed, double lo, double hi,
                         int64_t first_index, double *out) {
    /* inc/stencil.hpp:54-59 */
    if (n < 1) FAIL(ORC_INVALID_ARGUMENT, "vector length must be >= 1");
    for (int64_t i = 0; i < n; i++) {
        int64_t g = first_index + i;
        if (kind == 0) out[i] = 1.0;
        else if (kind == 1) out[i] = (double)g;
        else if (kind == 2) {
            double u = u01(h2(seed, (uint64_t)g));
            double w = (hi - lo) * u;
            out[i] = lo + w;
        } else FAIL(ORC_INVALID_ARGUMENT, "unknown vector kind %d", kind);
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* ELL                                                                        */
/* ------------------------------------------------------------------------- */
static int32_t csr_max_row(const orc_csr *m) {
    int32_t w = 0;
    for (int32_t i = 0; i < m->n; i++) {
        int32_t k = (int32_t)(m->row_start[i + 1] - m->row_start[i]);
        if (k > w) w = k;
    }
    return w;
}

int orc_to_ell(const orc_csr *m, int32_t min_width, int64_t row_offset, orc_ell **out) {
    /* inc/ell.hpp:10-13,28-29; width = max row nnz, real
     * entries keep ascending-column order, trailing padding = (0.0, own row).
     * min_width lets a chunk use the global width; row_offset is the global id
     * of local row 0 (padding column = own GLOBAL row). */
    orc_ell *a = calloc(1, sizeof *a);
    if (!a) FAIL(ORC_NOMEM, "out of memory");
    a->n = m->n;
    a->width = csr_max_row(m);
    if (a->width < min_width) a->width = min_width;
    a->nnz = m->row_start[m->n];
    a->row_offset = row_offset;
    size_t slots = (size_t)a->n * (size_t)a->width;
    a->values = malloc((slots + 1) * sizeof(double));
    a->columns = malloc((slots + 1) * sizeof(int32_t));
    if (!a->values || !a->columns) { orc_ell_free(a); FAIL(ORC_NOMEM, "out of memory"); }
    for (int32_t i = 0; i < a->n; i++) {
        int64_t b = m->row_start[i];
        int32_t k = (int32_t)(m->row_start[i + 1] - b);
        int64_t s = (int64_t)i * a->width; /* inc/ell.hpp:21-23 */
        for (int32_t t = 0; t < a->width; t++) {
            a->values[s + t] = t < k ? m->vals[b + t] : 0.0;
            a->columns[s + t] = t < k ? m->cols[b + t] : (int32_t)(row_offset + i);
        }
    }
    *out = a;
    return ORC_OK;
}

int orc_ell_to_csr(const orc_ell *a, orc_csr **out) {
    /* inc/ell.hpp:31-32: drop padding slots (value 0.0, column = own row) */
    orc_csr *m = calloc(1, sizeof *m);
    m->n = a->n;
    size_t slots = (size_t)a->n * (size_t)a->width;
    m->row_start = malloc((size_t)(a->n + 1) * sizeof(int64_t));
    m->cols = malloc((slots + 1) * sizeof(int32_t));
    m->vals = malloc((slots + 1) * sizeof(double));
    int64_t pos = 0;
    for (int32_t i = 0; i < a->n; i++) {
        m->row_start[i] = pos;
        int64_t s = (int64_t)i * a->width;
        for (int32_t t = 0; t < a->width; t++) {
            int32_t c = a->columns[s + t];
            double v = a->values[s + t];
            if (v == 0.0 && c == (int32_t)(a->row_offset + i)) continue; /* padding slot */
            m->cols[pos] = c;
            m->vals[pos] = v;
            pos++;
        }
    }
    m->row_start[a->n] = pos;
    *out = m;
    return ORC_OK;
}

void orc_ell_free(orc_ell *a) {
    if (!a) return;
    free(a->values); free(a->columns); free(a);
}

/* ------------------------------------------------------------------------- */
/* value table                                                                */
/* ------------------------------------------------------------------------- */
static int cmp_double_bits(const void *pa, const void *pb) {
    double a = *(const double *)pa, b = *(const double *)pb;
    if (a < b) return -1;
    if (a > b) return 1;
    uint64_t ua, ub;
    memcpy(&ua, &a, 8); memcpy(&ub, &b, 8);
    return ua < ub ? -1 : ua > ub;
}

/* Insert into a small sorted set of distinct bit patterns; returns -1 on overflow. */
typedef struct vset { double *v; int32_t m; size_t limit; } vset;
static int vset_add(vset *s, double x) {
    int32_t lo = 0, hi = s->m;
    while (lo < hi) {
        int32_t mid = (lo + hi) / 2;
        if (cmp_double_bits(&s->v[mid], &x) < 0) lo = mid + 1; else hi = mid;
    }
    if (lo < s->m && !memcmp(&s->v[lo], &x, 8)) return 0;
    if ((size_t)s->m >= s->limit) return -1;
    memmove(s->v + lo + 1, s->v + lo, (size_t)(s->m - lo) * sizeof(double));
    s->v[lo] = x;
    s->m++;
    return 0;
}
static int32_t vset_find(const double *tab, int32_t m, double x) {
    int32_t lo = 0, hi = m;
    while (lo < hi) {
        int32_t mid = (lo + hi) / 2;
        if (cmp_double_bits(&tab[mid], &x) < 0) lo = mid + 1; else hi = mid;
    }
    return (lo < m && !memcmp(&tab[lo], &x, 8)) ? lo : -1;
}

int orc_scan_value_table(const orc_csr *m, size_t limit, double *table, int32_t *m_out) {
    /* inc/compress.hpp:11-26,80; distinct values by
     * bit pattern, strictly ascending; more than `limit` -> TableOverflowError. */
    vset s = {malloc((limit + 1) * sizeof(double)), 0, limit};
    int64_t nnz = m->row_start[m->n];
    for (int64_t t = 0; t < nnz; t++)
        if (vset_add(&s, m->vals[t]) < 0) {
            free(s.v);
            FAIL(ORC_TABLE_OVERFLOW, "more than %zu distinct matrix values", limit);
        }
    memcpy(table, s.v, (size_t)s.m * sizeof(double));
    *m_out = s.m;
    free(s.v);
    return ORC_OK;
}

/* Sort one row by (value ascending, column ascending) and
 * produce exclusive group ends per table value. */
typedef struct ent { int32_t vi; int32_t col; } ent;
static int cmp_ent(const void *a, const void *b) {
    const ent *x = a, *y = b;
    if (x->vi != y->vi) return x->vi < y->vi ? -1 : 1;
    return x->col < y->col ? -1 : x->col > y->col;
}
static int sort_row(const double *table, int32_t m, int k, const int32_t *cols, const double *vals,
                    ent *e, int32_t *ends) {
    for (int t = 0; t < k; t++) {
        e[t].vi = vset_find(table, m, vals[t]);
        if (e[t].vi < 0) return -1;
        e[t].col = cols[t];
    }
    qsort(e, (size_t)k, sizeof(ent), cmp_ent);
    int idx = 0;
    for (int32_t g = 0; g < m; g++) {
        while (idx < k && e[idx].vi == g) idx++;
        ends[g] = idx;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* vt format                                                                  */
/* ------------------------------------------------------------------------- */
int orc_compress_values(const orc_csr *mtx, size_t limit, int32_t min_width, int64_t row_offset,
                        orc_vt **out) {
    /* inc/compress.hpp:28-46,82 */
    double *table = malloc((limit + 1) * sizeof(double));
    int32_t m = 0;
    int rc = orc_scan_value_table(mtx, limit, table, &m);
    if (rc) { free(table); return rc; }
    orc_vt *c = calloc(1, sizeof *c);
    c->n = mtx->n;
    c->m = m;
    c->width = csr_max_row(mtx);
    if (c->width < min_width) c->width = min_width;
    c->row_offset = row_offset;
    c->table = table;
    size_t slots = (size_t)c->n * (size_t)c->width;
    c->sorted_columns = malloc((slots + 1) * sizeof(int32_t));
    c->ends = malloc(((size_t)c->n * (size_t)m + 1) * sizeof(int32_t));
    ent *e = malloc((size_t)(c->width + 1) * sizeof(ent));
    for (int32_t i = 0; i < c->n; i++) {
        int64_t b = mtx->row_start[i];
        int k = (int)(mtx->row_start[i + 1] - b);
        sort_row(table, m, k, mtx->cols + b, mtx->vals + b, e, c->ends + (int64_t)i * m);
        int64_t s = (int64_t)i * c->width;
        for (int32_t t = 0; t < c->width; t++) /* padding = own row, never read (compress.hpp:33-34) */
            c->sorted_columns[s + t] = t < k ? e[t].col : (int32_t)(row_offset + i);
    }
    free(e);
    *out = c;
    return ORC_OK;
}

int orc_validate_vt(const orc_vt *c, int64_t n_cols) {
    /* inc/compress.hpp:92-94 */
    for (int32_t k = 1; k < c->m; k++)
        if (!(c->table[k - 1] < c->table[k])) FAIL(ORC_INTEGRITY, "value table not strictly ascending at %d", k);
    for (int32_t i = 0; i < c->n; i++) {
        const int32_t *en = c->ends + (int64_t)i * c->m;
        int32_t prev = 0;
        for (int32_t k = 0; k < c->m; k++) {
            if (en[k] < prev) FAIL(ORC_INTEGRITY, "row %d: ends not monotone", i);
            prev = en[k];
        }
        if (prev > c->width) FAIL(ORC_INTEGRITY, "row %d: ends exceed width", i);
        for (int32_t t = 0; t < prev; t++) {
            int32_t col = c->sorted_columns[(int64_t)i * c->width + t];
            if (col < 0 || col >= n_cols) FAIL(ORC_INTEGRITY, "row %d: column %d out of range", i, col);
        }
    }
    return ORC_OK;
}

static int cmp_colval(const void *a, const void *b) {
    const ent *x = a, *y = b; /* col in .col, value index in .vi */
    return x->col < y->col ? -1 : x->col > y->col;
}

int orc_decompress_vt(const orc_vt *c, orc_csr **out) {
    /* inc/compress.hpp:87-89: exact triples, columns re-sorted */
    int rc = orc_validate_vt(c, INT64_MAX);
    if (rc) return rc;
    orc_csr *m = calloc(1, sizeof *m);
    m->n = c->n;
    size_t slots = (size_t)c->n * (size_t)c->width;
    m->row_start = malloc((size_t)(c->n + 1) * sizeof(int64_t));
    m->cols = malloc((slots + 1) * sizeof(int32_t));
    m->vals = malloc((slots + 1) * sizeof(double));
    ent *e = malloc((size_t)(c->width + 1) * sizeof(ent));
    int64_t pos = 0;
    for (int32_t i = 0; i < c->n; i++) {
        m->row_start[i] = pos;
        const int32_t *en = c->ends + (int64_t)i * c->m;
        int idx = 0;
        for (int32_t k = 0; k < c->m; k++)
            for (; idx < en[k]; idx++) {
                e[idx].col = c->sorted_columns[(int64_t)i * c->width + idx];
                e[idx].vi = k;
            }
        qsort(e, (size_t)idx, sizeof(ent), cmp_colval);
        for (int t = 0; t < idx; t++) { m->cols[pos] = e[t].col; m->vals[pos] = c->table[e[t].vi]; pos++; }
    }
    m->row_start[c->n] = pos;
    free(e);
    *out = m;
    return ORC_OK;
}

void orc_vt_free(orc_vt *c) {
    if (!c) return;
    free(c->table); free(c->sorted_columns); free(c->ends); free(c);
}

/* ------------------------------------------------------------------------- */
/* pattern format                                                             */
/* ------------------------------------------------------------------------- */
/* Row-shape key = (nnz, displacement[], value bits[]) in ascending-column order.
 * Two rows share a key iff their (displacement, value) sets are identical, which
 * for a fixed global value table is exactly "displacement list and ends list
 * match" (inc/compress.hpp:48-51).  Exact compare, no hash-only
 * dedup ("no hashing collisions permitted"). */
typedef struct shape {
    int32_t k;
    int32_t disp[ORC_MAX_ROW];
    uint64_t bits[ORC_MAX_ROW];
} shape;

typedef struct shape_slot {
    int64_t key_off;  /* into arena (int32 words) ; -1 = empty */
    int64_t first_row;
    int64_t count;
} shape_slot;

typedef struct shape_map {
    shape_slot *slots;
    size_t cap, used;
    int32_t *arena; /* per key: k, disp[k], bits as 2*k words */
    size_t arena_len, arena_cap;
} shape_map;

static uint64_t shape_hash(const shape *s) {
    uint64_t h = 0xcbf29ce484222325ULL ^ (uint64_t)s->k;
    for (int t = 0; t < s->k; t++) {
        h = sm64(h ^ (uint64_t)(uint32_t)s->disp[t]);
        h = sm64(h ^ s->bits[t]);
    }
    return h;
}
static int shape_eq_arena(const shape_map *mp, int64_t off, const shape *s) {
    const int32_t *a = mp->arena + off;
    if (a[0] != s->k) return 0;
    if (memcmp(a + 1, s->disp, (size_t)s->k * 4)) return 0;
    return !memcmp(a + 1 + s->k, s->bits, (size_t)s->k * 8);
}
static void shape_map_init(shape_map *mp) {
    mp->cap = 1024; mp->used = 0;
    mp->slots = malloc(mp->cap * sizeof(shape_slot));
    for (size_t i = 0; i < mp->cap; i++) mp->slots[i].key_off = -1;
    mp->arena_cap = 1 << 16; mp->arena_len = 0;
    mp->arena = malloc(mp->arena_cap * sizeof(int32_t));
}
static void shape_map_free(shape_map *mp) { free(mp->slots); free(mp->arena); }
static shape_slot *shape_map_probe(shape_map *mp, const shape *s, uint64_t h) {
    size_t i = (size_t)h & (mp->cap - 1);
    for (;;) {
        shape_slot *sl = &mp->slots[i];
        if (sl->key_off < 0 || shape_eq_arena(mp, sl->key_off, s)) return sl;
        i = (i + 1) & (mp->cap - 1);
    }
}
static void shape_from_arena(const shape_map *mp, int64_t off, shape *s) {
    const int32_t *a = mp->arena + off;
    s->k = a[0];
    memcpy(s->disp, a + 1, (size_t)s->k * 4);
    memcpy(s->bits, a + 1 + s->k, (size_t)s->k * 8);
}
static shape_slot *shape_map_add(shape_map *mp, const shape *s, int64_t row) {
    if ((mp->used + 1) * 2 > mp->cap) { /* grow + rehash */
        size_t ocap = mp->cap;
        shape_slot *old = mp->slots;
        mp->cap *= 2;
        mp->slots = malloc(mp->cap * sizeof(shape_slot));
        for (size_t i = 0; i < mp->cap; i++) mp->slots[i].key_off = -1;
        shape tmp;
        for (size_t i = 0; i < ocap; i++)
            if (old[i].key_off >= 0) {
                shape_from_arena(mp, old[i].key_off, &tmp);
                *shape_map_probe(mp, &tmp, shape_hash(&tmp)) = old[i];
            }
        free(old);
    }
    shape_slot *sl = shape_map_probe(mp, s, shape_hash(s));
    if (sl->key_off < 0) {
        size_t need = 1 + (size_t)s->k * 3;
        if (mp->arena_len + need > mp->arena_cap) {
            while (mp->arena_len + need > mp->arena_cap) mp->arena_cap *= 2;
            mp->arena = realloc(mp->arena, mp->arena_cap * sizeof(int32_t));
        }
        int32_t *a = mp->arena + mp->arena_len;
        a[0] = s->k;
        memcpy(a + 1, s->disp, (size_t)s->k * 4);
        memcpy(a + 1 + s->k, s->bits, (size_t)s->k * 8);
        sl->key_off = (int64_t)mp->arena_len;
        sl->first_row = row;
        sl->count = 0;
        mp->arena_len += need;
        mp->used++;
    }
    sl->count++;
    return sl;
}

static void row_shape(int64_t row, int k, const int32_t *cols, const double *vals, shape *s) {
    s->k = k;
    for (int t = 0; t < k; t++) {
        s->disp[t] = (int32_t)((int64_t)cols[t] - row);
        memcpy(&s->bits[t], &vals[t], 8);
    }
}

typedef struct kept { int64_t first_row; int64_t count; int64_t key_off; int32_t id; } kept;
static int cmp_kept_freq(const void *a, const void *b) {
    const kept *x = a, *y = b;
    if (x->count != y->count) return x->count > y->count ? -1 : 1; /* most frequent first */
    return x->first_row < y->first_row ? -1 : x->first_row > y->first_row;
}
static int cmp_kept_first(const void *a, const void *b) {
    const kept *x = a, *y = b;
    return x->first_row < y->first_row ? -1 : x->first_row > y->first_row;
}

static int compress_patterns_gen(const rowgen *g, int64_t n, int64_t row_offset, int values_in_pattern,
                                 size_t limit, int32_t min_rows, int32_t dict_cap, orc_pattern **out) {
    if (min_rows < 1) min_rows = 1;
    shape_map mp;
    shape_map_init(&mp);
    int32_t cols[ORC_MAX_ROW];
    double vals[ORC_MAX_ROW];
    shape s;
    /* pass 1: count row shapes */
    for (int64_t i = 0; i < n; i++) {
        int k = rowgen_row(g, i, cols, vals);
        if (k > ORC_MAX_ROW) { shape_map_free(&mp); FAIL(ORC_INVALID_ARGUMENT, "row %lld longer than %d", (long long)i, ORC_MAX_ROW); }
        row_shape(row_offset + i, k, cols, vals, &s);
        shape_map_add(&mp, &s, i);
    }
    /* choose the dictionary: shapes used by >= min_rows rows; if more than
     * dict_cap qualify keep the most frequent (ties: earlier first occurrence). */
    kept *kp = malloc((mp.used + 1) * sizeof(kept));
    size_t nk = 0;
    for (size_t i = 0; i < mp.cap; i++)
        if (mp.slots[i].key_off >= 0 && mp.slots[i].count >= min_rows) {
            kp[nk].first_row = mp.slots[i].first_row;
            kp[nk].count = mp.slots[i].count;
            kp[nk].key_off = mp.slots[i].key_off;
            nk++;
        }
    if (dict_cap > 0 && nk > (size_t)dict_cap) {
        qsort(kp, nk, sizeof(kept), cmp_kept_freq);
        nk = (size_t)dict_cap;
    }
    /* pattern ids: first occurrence in ascending row order (UNPINNED choice (1)) */
    qsort(kp, nk, sizeof(kept), cmp_kept_first);
    /* mark kept slots with their id: reuse `count` sign trick via side table */
    int32_t *slot_id = malloc(mp.cap * sizeof(int32_t));
    for (size_t i = 0; i < mp.cap; i++) slot_id[i] = -1;
    for (size_t p = 0; p < nk; p++) {
        shape_from_arena(&mp, kp[p].key_off, &s);
        shape_slot *sl = shape_map_probe(&mp, &s, shape_hash(&s));
        slot_id[sl - mp.slots] = (int32_t)p;
    }
    /* value table over dictionary rows only (exception rows keep raw values) */
    vset vs = {malloc((limit + 1) * sizeof(double)), 0, limit};
    for (size_t p = 0; p < nk; p++) {
        shape_from_arena(&mp, kp[p].key_off, &s);
        for (int t = 0; t < s.k; t++) {
            double v;
            memcpy(&v, &s.bits[t], 8);
            if (vset_add(&vs, v) < 0) {
                free(vs.v); free(kp); free(slot_id); shape_map_free(&mp);
                FAIL(ORC_TABLE_OVERFLOW, "more than %zu distinct matrix values", limit);
            }
        }
    }
    orc_pattern *c = calloc(1, sizeof *c);
    c->n = (int32_t)n;
    c->row_offset = row_offset;
    c->m = vs.m;
    c->table = vs.v;
    c->n_patterns = (int32_t)nk;
    c->values_in_pattern = values_in_pattern;
    c->disp_offsets = malloc((nk + 1) * sizeof(int64_t));
    size_t total = 0;
    for (size_t p = 0; p < nk; p++) total += (size_t)mp.arena[kp[p].key_off];
    c->disp_flat = malloc((total + 1) * sizeof(int32_t));
    c->ends_flat = malloc((nk * (size_t)(c->m ? c->m : 1) + 1) * sizeof(int32_t));
    ent e[ORC_MAX_ROW];
    int64_t pos = 0;
    for (size_t p = 0; p < nk; p++) {
        shape_from_arena(&mp, kp[p].key_off, &s);
        double v[ORC_MAX_ROW];
        for (int t = 0; t < s.k; t++) memcpy(&v[t], &s.bits[t], 8);
        /* (value asc, displacement asc) == (value asc, column asc) for one row */
        sort_row(c->table, c->m, s.k, s.disp, v, e, c->ends_flat + p * (size_t)c->m);
        c->disp_offsets[p] = pos;
        for (int t = 0; t < s.k; t++) c->disp_flat[pos++] = e[t].col;
    }
    c->disp_offsets[nk] = pos;
    /* pass 2: per-row ids and the exception block */
    c->row_pattern = malloc((size_t)(n + 1) * sizeof(int32_t));
    int32_t n_exc = 0, w_exc = 0;
    for (int64_t i = 0; i < n; i++) {
        int k = rowgen_row(g, i, cols, vals);
        row_shape(row_offset + i, k, cols, vals, &s);
        shape_slot *sl = shape_map_probe(&mp, &s, shape_hash(&s));
        int32_t id = slot_id[sl - mp.slots];
        c->row_pattern[i] = id;
        if (id < 0) { n_exc++; if (k > w_exc) w_exc = k; }
    }
    c->n_exc = n_exc;
    c->w_exc = w_exc;
    size_t eslots = (size_t)n_exc * (size_t)w_exc;
    c->exc_rows = malloc(((size_t)n_exc + 1) * sizeof(int32_t));
    c->exc_values = malloc((eslots + 1) * sizeof(double));
    c->exc_columns = malloc((eslots + 1) * sizeof(int32_t));
    int32_t q = 0;
    for (int64_t i = 0; i < n && n_exc > 0; i++) {
        if (c->row_pattern[i] >= 0) continue;
        int k = rowgen_row(g, i, cols, vals);
        c->exc_rows[q] = (int32_t)i;
        for (int32_t t = 0; t < w_exc; t++) {
            c->exc_values[(int64_t)q * w_exc + t] = t < k ? vals[t] : 0.0;
            c->exc_columns[(int64_t)q * w_exc + t] = t < k ? cols[t] : (int32_t)(row_offset + i);
        }
        q++;
    }
    free(kp); free(slot_id); shape_map_free(&mp);
    *out = c;
    return ORC_OK;
}

int orc_compress_patterns(const orc_csr *m, int values_in_pattern, size_t limit,
                          int32_t min_pattern_rows, int32_t dict_cap, int64_t row_offset, orc_pattern **out) {
    rowgen g;
    memset(&g, 0, sizeof g);
    g.csr = m;
    g.n = m->n;
    return compress_patterns_gen(&g, m->n, row_offset, values_in_pattern, limit, min_pattern_rows, dict_cap, out);
}

int orc_compress_patterns_grid(int nx, int ny, int nz, double diagonal, double off_diagonal,
                               const orc_perturb *p, int values_in_pattern, size_t limit,
                               int32_t min_pattern_rows, int32_t dict_cap, orc_pattern **out) {
    int rc = check_grid(nx, ny, nz);
    if (rc) return rc;
    rowgen g = {nx, ny, nz, diagonal, off_diagonal, {0, 0, 0, 0}, (int64_t)nx * ny * nz, NULL};
    if (p && p->enabled) g.pert = *p;
    return compress_patterns_gen(&g, g.n, 0, values_in_pattern, limit, min_pattern_rows, dict_cap, out);
}

int orc_validate_pattern(const orc_pattern *c, int64_t n_cols) {
    /* inc/compress.hpp:92-95 */
    for (int32_t k = 1; k < c->m; k++)
        if (!(c->table[k - 1] < c->table[k])) FAIL(ORC_INTEGRITY, "value table not strictly ascending at %d", k);
    for (int32_t p = 0; p < c->n_patterns; p++) {
        int64_t len = c->disp_offsets[p + 1] - c->disp_offsets[p];
        int32_t prev = 0;
        for (int32_t k = 0; k < c->m; k++) {
            int32_t en = c->ends_flat[(int64_t)p * c->m + k];
            if (en < prev) FAIL(ORC_INTEGRITY, "pattern %d: ends not monotone", p);
            prev = en;
        }
        if (prev != len) FAIL(ORC_INTEGRITY, "pattern %d: last end %d != displacement count %lld", p, prev, (long long)len);
    }
    int32_t q = 0;
    for (int32_t i = 0; i < c->n; i++) {
        int32_t id = c->row_pattern[i];
        if (id == -1) {
            if (q >= c->n_exc || c->exc_rows[q] != i) FAIL(ORC_INTEGRITY, "row %d: exception list out of step", i);
            for (int32_t t = 0; t < c->w_exc; t++) {
                int32_t col = c->exc_columns[(int64_t)q * c->w_exc + t];
                if (col < 0 || col >= n_cols) FAIL(ORC_INTEGRITY, "exception row %d: column %d out of range", i, col);
            }
            q++;
            continue;
        }
        if (id < 0 || id >= c->n_patterns) FAIL(ORC_INTEGRITY, "row %d: pattern id %d out of range", i, id);
        for (int64_t t = c->disp_offsets[id]; t < c->disp_offsets[id + 1]; t++) {
            int64_t col = c->row_offset + i + c->disp_flat[t];
            if (col < 0 || col >= n_cols) FAIL(ORC_INTEGRITY, "row %d: column %lld out of range", i, (long long)col);
        }
    }
    if (q != c->n_exc) FAIL(ORC_INTEGRITY, "exception count mismatch");
    return ORC_OK;
}

int orc_decompress_pattern(const orc_pattern *c, orc_csr **out) {
    /* inc/compress.hpp:87-90: row i = {(i + disp, table[group])}, columns re-sorted */
    int rc = orc_validate_pattern(c, INT64_MAX);
    if (rc) return rc;
    orc_csr *m = calloc(1, sizeof *m);
    m->n = c->n;
    size_t cap = 0;
    for (int32_t i = 0; i < c->n; i++) {
        int32_t id = c->row_pattern[i];
        cap += id >= 0 ? (size_t)(c->disp_offsets[id + 1] - c->disp_offsets[id]) : (size_t)c->w_exc;
    }
    m->row_start = malloc((size_t)(c->n + 1) * sizeof(int64_t));
    m->cols = malloc((cap + 1) * sizeof(int32_t));
    m->vals = malloc((cap + 1) * sizeof(double));
    ent e[ORC_MAX_ROW];
    int64_t pos = 0;
    int32_t q = 0;
    for (int32_t i = 0; i < c->n; i++) {
        m->row_start[i] = pos;
        int32_t id = c->row_pattern[i];
        if (id < 0) { /* exception row: ELL slots, trailing padding dropped */
            for (int32_t t = 0; t < c->w_exc; t++) {
                int32_t col = c->exc_columns[(int64_t)q * c->w_exc + t];
                double v = c->exc_values[(int64_t)q * c->w_exc + t];
                if (v == 0.0 && col == (int32_t)(c->row_offset + i)) continue; /* padding slot */
                m->cols[pos] = col; m->vals[pos] = v; pos++;
            }
            q++;
            continue;
        }
        int64_t b = c->disp_offsets[id];
        int idx = 0;
        for (int32_t k = 0; k < c->m; k++)
            for (; idx < c->ends_flat[(int64_t)id * c->m + k]; idx++) {
                e[idx].col = (int32_t)(c->row_offset + i + c->disp_flat[b + idx]);
                e[idx].vi = k;
            }
        qsort(e, (size_t)idx, sizeof(ent), cmp_colval);
        for (int t = 0; t < idx; t++) { m->cols[pos] = e[t].col; m->vals[pos] = c->table[e[t].vi]; pos++; }
    }
    m->row_start[c->n] = pos;
    *out = m;
    return ORC_OK;
}

void orc_pattern_free(orc_pattern *c) {
    if (!c) return;
    free(c->table); free(c->disp_offsets); free(c->disp_flat); free(c->ends_flat);
    free(c->row_pattern); free(c->exc_rows); free(c->exc_values); free(c->exc_columns); free(c);
}

/* ------------------------------------------------------------------------- */
/* SpMV                                                                       */
/* ------------------------------------------------------------------------- */
static void ell_rows(const orc_ell *a, const double *x, int64_t x0, double *y, int32_t b, int32_t e) {
    /* SPEC.md:208-211, inc/kernels.hpp:19-20: slot order, overwrite */
    for (int32_t i = b; i < e; i++) {
        const double *v = a->values + (int64_t)i * a->width;
        const int32_t *c = a->columns + (int64_t)i * a->width;
        double acc = 0.0;
        for (int32_t k = 0; k < a->width; k++) {
            double prod = v[k] * x[(int64_t)c[k] - x0];
            acc = acc + prod;
        }
        y[i] = acc;
    }
}
static void vt_rows(const orc_vt *a, const double *x, int64_t x0, double *y, int32_t b, int32_t e) {
    /* SPEC.md:218-221, inc/kernels.hpp:20-22: sum x within each value group in
     * stored order, then one product per group in table order */
    for (int32_t i = b; i < e; i++) {
        const int32_t *s = a->sorted_columns + (int64_t)i * a->width;
        const int32_t *en = a->ends + (int64_t)i * a->m;
        double acc = 0.0;
        int32_t idx = 0;
        for (int32_t k = 0; k < a->m; k++) {
            double sum = 0.0;
            for (; idx < en[k]; idx++) sum = sum + x[(int64_t)s[idx] - x0];
            double prod = a->table[k] * sum;
            acc = acc + prod;
        }
        y[i] = acc;
    }
}
static void pattern_rows(const orc_pattern *a, const double *x, int64_t x0, double *y, int32_t b, int32_t e) {
    /* PAPER.md:797-813 (List 1), inc/kernels.hpp:22: per
     * element value*x in group order.  Exception rows (id -1): ELL slot order. */
    int32_t q = 0;
    if (a->n_exc > 0) { /* first exception row >= b */
        int32_t lo = 0, hi = a->n_exc;
        while (lo < hi) { int32_t mid = (lo + hi) / 2; if (a->exc_rows[mid] < b) lo = mid + 1; else hi = mid; }
        q = lo;
    }
    for (int32_t i = b; i < e; i++) {
        int32_t type = a->row_pattern[i];
        double acc = 0.0;
        if (type < 0) {
            const double *v = a->exc_values + (int64_t)q * a->w_exc;
            const int32_t *c = a->exc_columns + (int64_t)q * a->w_exc;
            for (int32_t k = 0; k < a->w_exc; k++) {
                double prod = v[k] * x[(int64_t)c[k] - x0];
                acc = acc + prod;
            }
            q++;
            y[i] = acc;
            continue;
        }
        const int32_t *d = a->disp_flat + a->disp_offsets[type];
        const int32_t *en = a->ends_flat + (int64_t)type * a->m;
        int64_t gi = a->row_offset + i;
        int32_t idx = 0;
        for (int32_t k = 0; k < a->m; k++) {
            const double a_ij = a->table[k];
            for (; idx < en[k]; idx++) {
                int64_t j = gi + d[idx];
                double prod = a_ij * x[j - x0];
                acc = acc + prod;
            }
        }
        y[i] = acc;
    }
}

typedef struct job {
    int fmt;
    const void *a;
    const double *x;
    int64_t x0;
    double *y;
    int32_t b, e;
} job;
static void *job_run(void *p) {
    job *j = p;
    if (j->fmt == 0) ell_rows(j->a, j->x, j->x0, j->y, j->b, j->e);
    else if (j->fmt == 1) vt_rows(j->a, j->x, j->x0, j->y, j->b, j->e);
    else pattern_rows(j->a, j->x, j->x0, j->y, j->b, j->e);
    return NULL;
}
static void run_threads(int fmt, const void *a, const double *x, int64_t x0, double *y,
                        int32_t b, int32_t e, int threads) {
    /* contiguous row ranges, one join */
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if ((int64_t)threads > (int64_t)e - b) threads = (e - b) > 0 ? (e - b) : 1;
    job jobs[256];
    pthread_t th[256];
    int64_t span = (int64_t)e - b;
    for (int t = 0; t < threads; t++) {
        jobs[t] = (job){fmt, a, x, x0, y, (int32_t)(b + span * t / threads), (int32_t)(b + span * (t + 1) / threads)};
        if (t > 0) pthread_create(&th[t], NULL, job_run, &jobs[t]);
    }
    job_run(&jobs[0]);
    for (int t = 1; t < threads; t++) pthread_join(th[t], NULL);
}
void orc_spmv_ell(const orc_ell *a, const double *x, int64_t x0, double *y, int32_t b, int32_t e, int th) {
    run_threads(0, a, x, x0, y, b, e, th);
}
void orc_spmv_vt(const orc_vt *a, const double *x, int64_t x0, double *y, int32_t b, int32_t e, int th) {
    run_threads(1, a, x, x0, y, b, e, th);
}
void orc_spmv_pattern(const orc_pattern *a, const double *x, int64_t x0, double *y, int32_t b, int32_t e, int th) {
    run_threads(2, a, x, x0, y, b, e, th);
}

void orc_spmv_csr(const orc_csr *a, const double *x, double *y) {
    for (int32_t i = 0; i < a->n; i++) {
        double acc = 0.0;
        for (int64_t t = a->row_start[i]; t < a->row_start[i + 1]; t++) {
            double prod = a->vals[t] * x[a->cols[t]];
            acc = acc + prod;
        }
        y[i] = acc;
    }
}
void orc_row_abs_scale(const orc_csr *a, const double *x, double *scale) {
    for (int32_t i = 0; i < a->n; i++) {
        double acc = 0.0;
        for (int64_t t = a->row_start[i]; t < a->row_start[i + 1]; t++) acc += fabs(a->vals[t] * x[a->cols[t]]);
        scale[i] = acc;
    }
}

/* ------------------------------------------------------------------------- */
/* CG caller                                                                  */
/* ------------------------------------------------------------------------- */
double orc_dot(const double *u, const double *v, int64_t n) {
    /* sequential accumulation, index ascending */
    double acc = 0.0;
    for (int64_t i = 0; i < n; i++) {
        double prod = u[i] * v[i];
        acc = acc + prod;
    }
    return acc;
}
void orc_waxpby(double alpha, const double *x, double beta, const double *y, double *w, int64_t n) {
    /* w[i] = alpha*x[i] + beta*y[i] */
    for (int64_t i = 0; i < n; i++) {
        double ax = alpha * x[i], by = beta * y[i];
        w[i] = ax + by;
    }
}
static void cg_spmv(int format, const void *a, int32_t n, const double *x, double *y) {
    if (format == 0) ell_rows(a, x, 0, y, 0, n);
    else if (format == 1) vt_rows(a, x, 0, y, 0, n);
    else pattern_rows(a, x, 0, y, 0, n);
}
int orc_cg_solve(int format, const void *a, int32_t n, const double *b, double *x, int32_t max_iterations,
                 double tolerance, int32_t *iterations, int32_t *converged, double *history, int32_t *diverged_at) {
    /* solver.hpp:40-46: r = b - A*0, z = r (no preconditioner), p = z; per iteration exactly
     * 1 SpMV, 3 dots, 3 waxpbys; stop when ||r||2 / ||b||2 <= tolerance. */
    if (max_iterations < 1 || !(tolerance > 0.0) || format < 0 || format > 2)
        FAIL(ORC_INVALID_ARGUMENT, "cg_solve: bad configuration");
    double *r = malloc((size_t)n * 8), *p = malloc((size_t)n * 8), *ap = malloc((size_t)n * 8);
    *iterations = 0; *converged = 0; *diverged_at = 0;
    for (int32_t i = 0; i < n; i++) { x[i] = 0.0; r[i] = b[i]; p[i] = b[i]; }
    double bnorm = sqrt(orc_dot(b, b, n));
    double rz = orc_dot(r, r, n);
    history[0] = 1.0;
    if (bnorm == 0.0) { *converged = 1; free(r); free(p); free(ap); return ORC_OK; }
    for (int32_t it = 1; it <= max_iterations; it++) {
        cg_spmv(format, a, n, p, ap);
        double alpha = rz / orc_dot(p, ap, n);
        orc_waxpby(1.0, x, alpha, p, x, n);
        orc_waxpby(1.0, r, -alpha, ap, r, n);
        double rr = orc_dot(r, r, n);
        double rz_new = orc_dot(r, r, n);
        double rel = sqrt(rr) / bnorm;
        *iterations = it;
        history[it] = rel;
        if (!isfinite(alpha) || !isfinite(rel)) { *diverged_at = it; break; }
        if (rel <= tolerance) { *converged = 1; break; }
        double beta = rz_new / rz;
        rz = rz_new;
        orc_waxpby(1.0, r, beta, p, p, n);
    }
    free(r); free(p); free(ap);
    return ORC_OK;
}

int orc_symgs_sweep(const orc_csr *m, double *x, const double *b) {
    /* kernels.hpp:44-48: one forward sweep (rows ascending) then one backward sweep (rows descending),
     * x[i] <- (b[i] - sum_{j != i} a_ij x[j]) / a_ii with the latest values; the sum runs over the row's entries in
     * ascending column order, every product and sum rounded separately. */
    for (int32_t i = 0; i < m->n; i++) {
        int found = 0;
        for (int64_t t = m->row_start[i]; t < m->row_start[i + 1]; t++)
            if (m->cols[t] == i && m->vals[t] != 0.0) found = 1;
        if (!found) FAIL(ORC_INVALID_ARGUMENT, "symgs_sweep: zero or missing diagonal in row %d (singular)", i);
    }
    for (int dir = 0; dir < 2; dir++)
        for (int32_t k = 0; k < m->n; k++) {
            const int32_t i = dir == 0 ? k : m->n - 1 - k;
            double sum = 0.0, diag = 0.0;
            for (int64_t t = m->row_start[i]; t < m->row_start[i + 1]; t++) {
                if (m->cols[t] == i) diag = m->vals[t];
                else sum = sum + m->vals[t] * x[m->cols[t]];
            }
            x[i] = (b[i] - sum) / diag;
        }
    return ORC_OK;
}

int orc_pcg_solve(int format, const void *a, const orc_csr *m, int32_t n, const double *b, double *x, int32_t max_iterations,
                  double tolerance, int32_t sweeps, int32_t *iterations, int32_t *converged, double *history, int32_t *diverged_at) {
    /* solver.hpp:40-46, SPEC.md:308-311 with the SymGS preconditioner: z <- M^-1 r = `sweeps` symgs_sweep calls on A z = r
     * from a zero initial guess; per iteration 1 SpMV, 3 dots (p.Ap, r.r, r.z), 3 waxpbys, 1 preconditioner application. */
    if (max_iterations < 1 || !(tolerance > 0.0) || format < 0 || format > 2 || sweeps < 1 || m->n != n)
        FAIL(ORC_INVALID_ARGUMENT, "pcg_solve: bad configuration");
    double *r = malloc((size_t)n * 8), *z = malloc((size_t)n * 8), *p = malloc((size_t)n * 8), *ap = malloc((size_t)n * 8);
    int rc = ORC_OK;
    *iterations = 0; *converged = 0; *diverged_at = 0;
    for (int32_t i = 0; i < n; i++) { x[i] = 0.0; r[i] = b[i]; z[i] = 0.0; }
    for (int32_t s = 0; s < sweeps && rc == ORC_OK; s++) rc = orc_symgs_sweep(m, z, r);
    if (rc != ORC_OK) { free(r); free(z); free(p); free(ap); return rc; }
    for (int32_t i = 0; i < n; i++) p[i] = z[i];
    double bnorm = sqrt(orc_dot(b, b, n));
    double rz = orc_dot(r, z, n);
    history[0] = 1.0;
    if (bnorm == 0.0) { *converged = 1; free(r); free(z); free(p); free(ap); return ORC_OK; }
    for (int32_t it = 1; it <= max_iterations; it++) {
        cg_spmv(format, a, n, p, ap);
        double alpha = rz / orc_dot(p, ap, n);
        orc_waxpby(1.0, x, alpha, p, x, n);
        orc_waxpby(1.0, r, -alpha, ap, r, n);
        double rr = orc_dot(r, r, n);
        double rel = sqrt(rr) / bnorm;
        *iterations = it;
        history[it] = rel;
        if (!isfinite(alpha) || !isfinite(rel)) { *diverged_at = it; break; }
        if (rel <= tolerance) { *converged = 1; break; }
        for (int32_t i = 0; i < n; i++) z[i] = 0.0;
        for (int32_t s = 0; s < sweeps; s++) orc_symgs_sweep(m, z, r);
        double rz_new = orc_dot(r, z, n);
        double beta = rz_new / rz;
        rz = rz_new;
        orc_waxpby(1.0, z, beta, p, p, n);
    }
    free(r); free(z); free(p); free(ap);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* byte model                                                                 */
/* ------------------------------------------------------------------------- */
static void cost_finish(orc_cost *c, double flops_per_row) {
    c->bytes_per_row = c->values + c->indices + c->ends + c->pattern_id + c->input_vector;
    c->flops_per_row = flops_per_row;
    c->bytes_per_flop = flops_per_row > 0 ? c->bytes_per_row / flops_per_row : 0.0;
}
int orc_format_cost(int format, int row_nnz, int table_size, int include_x, orc_cost *c) {
    /* inc/perf_model.hpp:49-57 */
    memset(c, 0, sizeof *c);
    switch (format) {
    case 0: c->values = 8.0 * row_nnz; c->indices = 4.0 * row_nnz; break;
    case 1: c->indices = 4.0 * row_nnz; c->ends = 4.0 * table_size; break;
    case 2: c->pattern_id = 4.0; c->ends = 4.0 * table_size; break;
    case 3: c->pattern_id = 4.0; break;
    default: FAIL(ORC_INVALID_ARGUMENT, "unknown format %d", format);
    }
    if (include_x) c->input_vector = 8.0; /* inc/perf_model.hpp:42-47 */
    cost_finish(c, 2.0 * row_nnz);
    return ORC_OK;
}
double orc_required_bandwidth(double flops_per_second, const orc_cost *c) {
    return flops_per_second * c->bytes_per_flop; /* inc/perf_model.hpp:59-60 */
}
double orc_roofline(const orc_cost *c, double bw, double peak, int *limiting) {
    /* inc/perf_model.hpp:71-72 */
    double f = bw / c->bytes_per_flop;
    int lim = 0;
    if (peak > 0 && peak < f) { f = peak; lim = 1; }
    if (limiting) *limiting = lim;
    return f;
}
int orc_measured_cost_ell(const orc_ell *a, orc_cost *c) {
    /* inc/perf_model.hpp:74-78: bytes the kernel streams per row */
    memset(c, 0, sizeof *c);
    c->values = 8.0 * a->width;
    c->indices = 4.0 * a->width;
    cost_finish(c, 2.0 * (double)a->nnz / a->n);
    return ORC_OK;
}
int orc_measured_cost_vt(const orc_vt *a, orc_cost *c) {
    memset(c, 0, sizeof *c);
    int64_t nnz = 0;
    for (int32_t i = 0; i < a->n; i++) nnz += a->ends[(int64_t)(i + 1) * a->m - 1];
    c->indices = 4.0 * a->width;
    c->ends = 4.0 * a->m;
    cost_finish(c, 2.0 * (double)nnz / a->n);
    return ORC_OK;
}
int orc_measured_cost_pattern(const orc_pattern *a, orc_cost *c) {
    /* per-row ids, plus the pattern tables amortised over rows; with
     * values_in_pattern == 0 the group ends are charged per row
     * (inc/compress.hpp:60-64, inc/perf_model.hpp:74-77).  Exception rows add
     * their ELL slots and their row index (extension). */
    memset(c, 0, sizeof *c);
    int64_t nnz = 0;
    for (int32_t i = 0; i < a->n; i++) {
        int32_t id = a->row_pattern[i];
        if (id >= 0) nnz += a->disp_offsets[id + 1] - a->disp_offsets[id];
    }
    for (int64_t t = 0; t < (int64_t)a->n_exc * a->w_exc; t++)
        if (!(a->exc_values[t] == 0.0)) nnz++;
    double n = a->n;
    c->pattern_id = 4.0;
    c->indices = 4.0 * (double)a->disp_offsets[a->n_patterns] / n + (4.0 * a->w_exc + 4.0) * a->n_exc / n;
    c->values = 8.0 * (double)a->w_exc * a->n_exc / n;
    c->ends = a->values_in_pattern ? 4.0 * a->m * a->n_patterns / n : 4.0 * a->m;
    cost_finish(c, 2.0 * (double)nnz / n);
    return ORC_OK;
}
