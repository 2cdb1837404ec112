/*
 * spmvcomp_oracle.h -- CPU ORACLE (TEST INFRASTRUCTURE, NOT PRODUCT CODE).
 *
 * A plain-C restatement of the reference library `spmvcomp` (arxiv 1612.00530)
 * for the SpMV hot path: generator, ELL / value-table / pattern formats,
 * decompression, validation, the three SpMV kernels and the byte model.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product (the CUDA library
 * under paper_1612_00530_b200/csrc) never links, loads or calls it.
 *
 * The reference ships declarations only (no src/): every body here is restated
 * from /root/reference/SPEC.md, the headers under proj/include/spmvcomp and
 * PAPER.md List 1.  Each function cites the lines it follows.
 *
 * PINNED by the reference's own worked examples / known answers (tests/test_oracle_kat.py):
 *   generator K1-K3,K15; figure row K4; pattern count K5; value table K6;
 *   ELL K7; 1x1 SpMV K8; A*ones K9; dense product K10,K11; round trip K12;
 *   byte model K13,K14.  (SURVEY.md section 8c.)
 * PARITY UNPINNED (nothing in the reference fixes these; choices made here and
 * mirrored by the product, documented in DESIGN.md):
 *   (1) pattern-id numbering = first occurrence in ascending row order;
 *   (2) the random-vector generator (counter-based splitmix64, value i depends
 *       only on (seed, i));  (3) the [lo,hi) range extension of make_test_vector;
 *   (4) exception rows (hybrid format) and the config-4 perturbation recipe;
 *   (5) relative-error scale when y_ref == 0.
 * Floating point: compile with -ffp-contract=off and no -march flag, i.e. the
 * arithmetic the reference's own CMake Release build (g++ -O3, baseline x86-64,
 * no FMA instruction available) would perform for `y[i] += a_ij * x_j`.
 */
#ifndef SPMVCOMP_ORACLE_H
#define SPMVCOMP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: mirror errors.hpp:9-42 plus std::invalid_argument */
enum {
    ORC_OK = 0,
    ORC_INVALID_ARGUMENT = 1, /* grid.hpp:35-47, length mismatch SPEC.md:212 */
    ORC_TABLE_OVERFLOW = 2,   /* errors.hpp:9  */
    ORC_INTEGRITY = 3,        /* errors.hpp:16 */
    ORC_NOMEM = 9
};

const char *orc_last_error(void);

/* ---- CSR (StencilMatrix, stencil.hpp:19-36) ------------------------------ */
typedef struct orc_csr {
    int32_t n;
    int64_t *row_start; /* n+1 */
    int32_t *cols;      /* nnz, strictly ascending per row */
    double *vals;       /* nnz */
    int32_t nx, ny, nz; /* provenance, 0 = unknown */
} orc_csr;

/* Perturbation recipe of BASELINE.json configs[3] (extension). */
typedef struct orc_perturb {
    int enabled;
    uint64_t seed;   /* seed_p, 11 in the config */
    double fraction; /* 0.1 */
    double noise;    /* 0.1 -> off-diagonals get U[-0.1,0.1) added */
} orc_perturb;

/* generate_matrix (stencil.hpp:40-45), rows [row_begin,row_end)
 * of the global grid; columns are global.  row_begin=0,row_end=n gives the
 * whole matrix.  `p` may be NULL (no perturbation). */
int orc_generate_rows(int nx, int ny, int nz, double diagonal, double off_diagonal,
                      const orc_perturb *p, int64_t row_begin, int64_t row_end, orc_csr **out);
/* stencil_from_rows (stencil.hpp:47-50): validating copy of explicit CSR. */
int orc_csr_from_arrays(int32_t n, const int64_t *row_start, const int32_t *cols,
                        const double *vals, orc_csr **out);
void orc_csr_free(orc_csr *m);
int orc_csr_equal(const orc_csr *a, const orc_csr *b); /* stencil.hpp:38 */
int orc_is_symmetric(const orc_csr *m);                /* stencil.hpp:52 */

/* make_test_vector (stencil.hpp:54-59). kind: 0 ones, 1 linear,
 * 2 random in [lo,hi).  Element i of the random kind depends only on
 * (seed, first_index + i) so slabs agree with the global vector. */
int orc_make_test_vector(int64_t n, int kind, uint64_t seed, double lo, double hi,
                         int64_t first_index, double *out);

/* ---- ELL (ell.hpp:10-32) -------------------------------------------------- */
typedef struct orc_ell {
    int32_t n, width;
    int64_t nnz;
    int64_t row_offset; /* global index of local row 0 (0 unless built from a chunk) */
    double *values;     /* n*width */
    int32_t *columns;   /* n*width */
} orc_ell;
int orc_to_ell(const orc_csr *m, int32_t min_width, int64_t row_offset, orc_ell **out);
int orc_ell_to_csr(const orc_ell *a, orc_csr **out); /* to_stencil, ell.hpp:31-32 */
void orc_ell_free(orc_ell *a);

/* ---- value table (compress.hpp:11-20,80) ---------------------------------- */
int orc_scan_value_table(const orc_csr *m, size_t limit, double *table, int32_t *m_out);

/* ---- vt format (compress.hpp:28-46,82) ------------------------------------ */
typedef struct orc_vt {
    int32_t n, width, m;
    int64_t row_offset;
    double *table;           /* m */
    int32_t *sorted_columns; /* n*width */
    int32_t *ends;           /* n*m */
} orc_vt;
int orc_compress_values(const orc_csr *m, size_t limit, int32_t min_width, int64_t row_offset,
                        orc_vt **out);
int orc_validate_vt(const orc_vt *c, int64_t n_cols);       /* compress.hpp:92-94 */
int orc_decompress_vt(const orc_vt *c, orc_csr **out);      /* compress.hpp:87-89 */
void orc_vt_free(orc_vt *c);

/* ---- pattern format (compress.hpp:48-85) + exception rows (extension H) --- */
typedef struct orc_pattern {
    int32_t n, m;
    int64_t row_offset;
    double *table;        /* m */
    int32_t n_patterns;
    int64_t *disp_offsets; /* n_patterns+1 offsets into disp_flat */
    int32_t *disp_flat;    /* displacements, (value asc, disp asc) order */
    int32_t *ends_flat;    /* n_patterns*m exclusive group ends */
    int32_t *row_pattern;  /* n ids; -1 marks an exception row */
    int values_in_pattern;
    /* exception block: uncompressed ELL rows for ids == -1 (extension) */
    int32_t n_exc, w_exc;
    int32_t *exc_rows;    /* ascending LOCAL row ids */
    double *exc_values;   /* n_exc*w_exc */
    int32_t *exc_columns; /* n_exc*w_exc, global columns; padding = own global row */
} orc_pattern;

/* compress_patterns (compress.hpp:84): min_pattern_rows=1, dict_cap=0 (none)
 * reproduces the reference scheme (every row gets an id, no exceptions).
 * min_pattern_rows>=2 activates the hybrid rule of DESIGN.md: a full
 * (displacement,value) row shape enters the dictionary iff at least that many
 * rows use it; all other rows become exception rows.  row_offset = global id of
 * the CSR's row 0 when it is a slab of a larger matrix (displacements are taken
 * against the GLOBAL row index). */
int orc_compress_patterns(const orc_csr *m, int values_in_pattern, size_t limit,
                          int32_t min_pattern_rows, int32_t dict_cap, int64_t row_offset, orc_pattern **out);
/* Same result as orc_generate_rows(whole grid) + orc_compress_patterns, but
 * streams the rows through the deduplicator without materialising the CSR
 * (for 256^3 and above). */
int orc_compress_patterns_grid(int nx, int ny, int nz, double diagonal, double off_diagonal,
                               const orc_perturb *p, int values_in_pattern, size_t limit,
                               int32_t min_pattern_rows, int32_t dict_cap, orc_pattern **out);
int orc_validate_pattern(const orc_pattern *c, int64_t n_cols);
int orc_decompress_pattern(const orc_pattern *c, orc_csr **out);
void orc_pattern_free(orc_pattern *c);

/* ---- SpMV (kernels.hpp:19-36) ----------
 * Local rows [begin,end); x is indexed by (global column - x_col0); y by local
 * row.  Overwrite semantics.  threads>1 splits [begin,end) into contiguous
 * ranges; results are bit-identical for any partition. */
void orc_spmv_ell(const orc_ell *a, const double *x, int64_t x_col0, double *y,
                  int32_t begin, int32_t end, int threads);
void orc_spmv_vt(const orc_vt *a, const double *x, int64_t x_col0, double *y,
                 int32_t begin, int32_t end, int threads);
void orc_spmv_pattern(const orc_pattern *a, const double *x, int64_t x_col0, double *y,
                      int32_t begin, int32_t end, int threads);
/* CSR product, ascending column order: the brute-force cross-check of SPEC.md:216,269. */
void orc_spmv_csr(const orc_csr *a, const double *x, double *y);
/* sum_k |a_ik * x_k| per row: the scale for "relative per row". */
void orc_row_abs_scale(const orc_csr *a, const double *x, double *scale);

/* ---- CG caller (kernels.hpp:39-42, solver.hpp:40-46) -- */
double orc_dot(const double *u, const double *v, int64_t n);                 /* index-ascending sum */
void orc_waxpby(double alpha, const double *x, double beta, const double *y, double *w, int64_t n);
/* Unpreconditioned CG, x0 = 0.  format: 0 ell, 1 vt, 2 pattern (the SpMV backend); `a` points
 * to the matching struct.  history needs max_iterations+1 slots.  Returns ORC_OK, or
 * ORC_INVALID_ARGUMENT; *diverged_at > 0 when a non-finite value appeared. */
int orc_cg_solve(int format, const void *a, int32_t n, const double *b, double *x, int32_t max_iterations,
                 double tolerance, int32_t *iterations, int32_t *converged, double *history, int32_t *diverged_at);

/* symgs_sweep (kernels.hpp:44-48): forward then backward Gauss-Seidel in natural order, in place;
 * ORC_INVALID_ARGUMENT for a zero or missing diagonal ("singularity error"). */
int orc_symgs_sweep(const orc_csr *m, double *x, const double *b);
/* CG with the SymGS preconditioner (z = `sweeps` sweeps from a zero guess); m = the matrix as CSR. */
int orc_pcg_solve(int format, const void *a, const orc_csr *m, int32_t n, const double *b, double *x, int32_t max_iterations,
                  double tolerance, int32_t sweeps, int32_t *iterations, int32_t *converged, double *history, int32_t *diverged_at);

/* ---- byte model (perf_model.hpp:49-80) -------------------- */
typedef struct orc_cost {
    double bytes_per_row, flops_per_row, bytes_per_flop;
    double values, indices, ends, pattern_id, input_vector;
} orc_cost;
/* format: 0 ell, 1 vt, 2 pattern, 3 pattern_with_values (perf_model.hpp:14) */
int orc_format_cost(int format, int row_nnz, int table_size, int include_input_vector,
                    orc_cost *out);
double orc_required_bandwidth(double flops_per_second, const orc_cost *c);
/* returns predicted flops; *limiting = 0 bandwidth, 1 compute. peak_flops<=0 = absent */
double orc_roofline(const orc_cost *c, double read_bandwidth, double peak_flops, int *limiting);
int orc_measured_cost_ell(const orc_ell *a, orc_cost *out);
int orc_measured_cost_vt(const orc_vt *a, orc_cost *out);
int orc_measured_cost_pattern(const orc_pattern *a, orc_cost *out);

#ifdef __cplusplus
}
#endif
#endif
