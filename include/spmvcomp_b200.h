/*
 * spmvcomp_b200.h -- C-ABI of the B200-native SpMV path of `spmvcomp`
 * (arxiv 1612.00530).  This is the drop-in boundary: plain pointers and sizes,
 * no C++ or torch types.  Every entry point returns an int status (0 = ok);
 * no exception crosses the boundary; spmvb_last_error() gives the message of
 * the calling thread's last failure.
 *
 * Each entry point names the reference interface it stands in for, as
 * file:line under /root/reference/proj/include/spmvcomp (abbreviated inc/).
 * The C++ header set in include/spmvcomp/ implements the reference's C++ API
 * on top of these calls; INTEGRATION.md shows the binding a maintainer adds.
 *
 * Threading: one host thread drives a handle; calls on one handle are not
 * re-entrant; distinct handles are independent.  All device work is issued on
 * the caller's stream (a cudaStream_t passed as void*; NULL = default stream).
 * There is NO CPU fallback: without a CUDA device every compute entry point
 * fails with SPMVB_ERR_CUDA.
 */
#ifndef SPMVCOMP_B200_H
#define SPMVCOMP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: 1:1 with the reference's exception taxonomy (inc/errors.hpp:9-42,
 * std::invalid_argument from inc/grid.hpp:35-47) plus CUDA / NCCL / memory. */
enum spmvb_status {
    SPMVB_OK = 0,
    SPMVB_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    SPMVB_ERR_TABLE_OVERFLOW = 2,   /* TableOverflowError  inc/errors.hpp:9  */
    SPMVB_ERR_INTEGRITY = 3,        /* IntegrityError      inc/errors.hpp:16 */
    SPMVB_ERR_VERIFICATION = 4,     /* VerificationError   inc/errors.hpp:33 */
    SPMVB_ERR_IO = 5,               /* IoError             inc/errors.hpp:39 */
    SPMVB_ERR_DIVERGENCE = 6,       /* DivergenceError     inc/errors.hpp:22 */
    SPMVB_ERR_CUDA = 7,
    SPMVB_ERR_NCCL = 8,
    SPMVB_ERR_NOMEM = 9
};

/* inc/perf_model.hpp:14 MatrixFormat (pattern_with_values is the same device
 * structure as pattern with values_in_pattern set, inc/compress.hpp:60-64). */
enum spmvb_format { SPMVB_FMT_ELL = 0, SPMVB_FMT_VT = 1, SPMVB_FMT_PATTERN = 2, SPMVB_FMT_CSR = 3 };

/* Device arrays of a matrix handle; names follow the reference structs
 * (inc/ell.hpp:14-24, inc/compress.hpp:35-44,65-76, inc/stencil.hpp:19-36). */
enum spmvb_stream_id {
    SPMVB_S_VALUES = 0,          /* EllMatrix::values            f64  n*width      */
    SPMVB_S_COLUMNS = 1,         /* EllMatrix::columns           i32  n*width      */
    SPMVB_S_TABLE = 2,           /* ValueTable::entries          f64  m            */
    SPMVB_S_SORTED_COLUMNS = 3,  /* VtCompressedMatrix::sorted_columns i32 n*width */
    SPMVB_S_ENDS = 4,            /* VtCompressedMatrix::ends     i32  n*m          */
    SPMVB_S_ROW_PATTERN = 5,     /* PatternCompressedMatrix::row_pattern i32 n     */
    SPMVB_S_DISP_OFFSETS = 6,    /* offsets of patterns[p].displacements i64 P+1   */
    SPMVB_S_DISP_FLAT = 7,       /* patterns[p].displacements concatenated i32     */
    SPMVB_S_ENDS_FLAT = 8,       /* patterns[p].ends concatenated  i32 P*m         */
    SPMVB_S_EXC_ROWS = 9,        /* exception rows (extension)   i32  n_exc        */
    SPMVB_S_EXC_VALUES = 10,     /* exception ELL values         f64  n_exc*w_exc  */
    SPMVB_S_EXC_COLUMNS = 11,    /* exception ELL columns        i32  n_exc*w_exc  */
    SPMVB_S_CSR_ROW_START = 12,  /* StencilMatrix::row_start     i64  n+1          */
    SPMVB_S_CSR_COLS = 13,       /* StencilMatrix::cols          i32  nnz          */
    SPMVB_S_CSR_VALS = 14,       /* StencilMatrix::vals          f64  nnz          */
    SPMVB_S_COUNT_ = 15
};

typedef struct spmvb_matrix spmvb_matrix; /* opaque, device-resident, caller-destroyed */

typedef struct spmvb_matrix_info {
    int32_t format;            /* spmvb_format */
    int32_t n;                 /* local rows */
    int32_t width;             /* ELL / vt slot width */
    int32_t m;                 /* value-table size */
    int32_t n_patterns;
    int32_t n_exc, w_exc;      /* exception block */
    int32_t values_in_pattern;
    int64_t nnz;               /* real entries */
    int64_t row_offset;        /* global id of local row 0 (z-slab support) */
    int64_t disp_total;        /* total displacement count over all patterns */
    int32_t device;
    int32_t kernel_plan;       /* 0 generic, 1 sliding-window box plan (pattern format) */
    int32_t box_stride_y, box_stride_z; /* strides found in the dictionary (plan 1) */
    int32_t reserved_;
} spmvb_matrix_info;

/* Stencil grid + optional config-4 perturbation. */
typedef struct spmvb_grid {
    int32_t nx, ny, nz;        /* inc/grid.hpp:15-19 (GLOBAL grid) */
    double diagonal;           /* inc/stencil.hpp:44 default 26.0 */
    double off_diagonal;       /* inc/stencil.hpp:45 default -1.0 */
    int32_t perturb;           /* 0 = pure stencil */
    uint64_t perturb_seed;
    double perturb_fraction;   /* 0.1 */
    double perturb_noise;      /* 0.1 */
} spmvb_grid;

/* inc/compress.hpp:22-26 CompressOptions + the hybrid (exception-row) rule. */
typedef struct spmvb_compress_options {
    uint64_t value_table_limit; /* default 256 */
    int32_t values_in_pattern;  /* inc/compress.hpp:84 */
    int32_t min_pattern_rows;   /* 1 = reference scheme; >=2 = exception rows enabled */
    int32_t dict_cap;           /* 0 = unlimited */
} spmvb_compress_options;

/* ---- library / device ------------------------------------------------------ */
const char *spmvb_last_error(void);
int spmvb_version(void);
int spmvb_device_count(int *count);
int spmvb_set_device(int device);
/* Tuning knobs for A/B measurement, per host thread.  SpMV results never depend on them (every kernel keeps the format's
 * summation order); the one knob that touches floating-point results is "cg_fused_dot", which changes the order in which
 * p.Ap is summed inside spmvb_cg_solve (iterates then agree to rounding, iteration counts are unchanged in every test).
 * Unknown keys -> SPMVB_ERR_INVALID_ARGUMENT; so are values that select measurement-only variants unless the library
 * was built with -DSPMVB_LAB ("lab_build", read-only, says which; the default build holds none of them).
 *   "pattern_kernel": 0 auto, 1 List 1 as written (thread per row), 2 box plan required, 3 one-column box kernel only
 *   "box_march":      0 auto (tensor ring for ranges of >= 8 planes, else the register sliding window);
 *                     3 sliding window forced; 90 tensor ring forced, 101 / 107 / 108 / 109 / 110 / 111 / 112 its other schedules
 *                     (chunk per warp, ids by loads, round-robin tiles per CTA / per warp, 4 planes per thread, two lines per
 *                     step in chunks / in tiles);
 *                     lab build only: further variants and ablations (csrc/spmv_pattern*.cu list them with their times)
 *   "box_lines":      lines per CTA tile / chunk length of the tensor ring (0 = default)
 *   "exception_kernel": hybrid handles, the exception-row block: 0 / 1 (default) the ELL kernel with a row map, all gathers of a
 *                     row requested in one batch; 64 / 32: the rows' operands come from three shared-memory windows of x per
 *                     64- / 32-row tile (csrc/spmv_exception.cu; measured slower on BASELINE config 4: 43 vs 34 us; compiled into
 *                     lab builds only -- the default build runs the ELL kernel whatever the value)
 *   "exception_carveout": hybrid handles, the exception-block kernel's preferred shared-memory carve-out in percent of the SM's
 *                     228 KB (0 = default 60, -1 = the driver's choice): fewer CTAs per SM, more L1 for the scattered gathers
 *   "exception_overlap": hybrid handles: 1 (default) the exception block runs on a second stream beside the kernel of the dictionary
 *                     rows (the two write disjoint rows of y; forked and joined by events, so the call still completes in
 *                     stream order); 0 one after the other
 *   "ring_min_steps": tensor ring: fewest line steps per chunk before the grid shrinks below a full wave of CTAs (0 = default 4)
 *   "ring_two_lines": 1 (default) where x is far beyond L2 and the 64-column strips come in fours, a step of the tensor ring sums
 *                     the rows of two lines (4 planes x 2 lines x 2 columns per thread, tiles of 28 lines): 512^3 584 -> 546 us;
 *                     0 one line per step there as everywhere else
 *   "ring_pdl":       1 (default) the tensor-ring kernel is launched with programmatic stream serialization: its CTAs take the
 *                     places of the previous kernel's CTAs as those exit and wait (griddepcontrol.wait) for that kernel to
 *                     complete before touching global memory; 0 plain stream order
 *   "ring_leftover":  tensor ring, the one column past the last 64-column strip when 64 divides the line length: 0 (default)
 *                     its operands travel in the last strip's shared-memory ring; in the chunk-per-CTA kernels that warp sets
 *                     them aside per line and the whole CTA sums the column's rows at the end of a march (256^3: 66.7 -> 65.9 us,
 *                     512^3: 596 -> 582 us), in the chunk-per-warp kernels the warp sums them step by step; 2 step by step
 *                     everywhere; 1 row by row from global memory after the marches (the round-1 scheme; 256^3: 73.7 us)
 *   "host_chunks":    row chunks of the pipelined spmvb_spmv_host (0 = default 8)
 *   "host_stage":     1 (default) spmvb_spmv_host moves PAGEABLE host vectors through process-wide pinned bounce buffers, filled and
 *                     drained by "host_copy_threads" host threads (0 = default 8) inside the same chunk pipeline; 0 leaves them to
 *                     the driver's pageable copies.  Pinned (or registered) buffers are used in place either way
 *   "slab_graph":     1 (default) spmvb_slab_spmv replays its copies and launches as a CUDA graph; 0 launches directly
 *   "symgs_pipeline": 1 (default) a symgs sweep of a matrix whose rows are sub-boxes of the 27-point stencil (lines of at most 256
 *                     nodes) runs as a pipeline of planes: a CTA per plane, operands through shared-memory rings, release / acquire
 *                     clocks between neighbouring planes (256^3: 25.3 -> 14.9 ms per sweep); 0 never.  "symgs_lag": steps a plane
 *                     trails the one below (>= 5; 0 = 5).  "last_symgs_kernel" (read-only): 2 the pipeline, 1 the grid-barrier
 *                     kernel, 0 a launch per level.  Same bits whichever runs
 *   "symgs_persistent": 1 (default) a symgs sweep is ONE cooperative launch: a CTA per SM walks the hyperplane levels with a
 *                     grid-wide barrier between them and fetches each row's matrix data ahead of the barrier; 0 a launch
 *                     per level (recorded into a CUDA graph when "symgs_graph" = 1).  Same bits either way
 *   "symgs_graph":    1 (default) the launches of a symgs sweep are recorded into a CUDA graph and replayed; 0 launches directly
 *   "cg_graph":       1 (default) spmvb_cg_solve records its iteration into a CUDA graph after the first one and replays it (one
 *                     graph launch per iteration); 0 launches the kernels directly.  "last_cg_graph" (read-only) says which ran
 *   "cg_fused_scalars": spmvb_cg_solve's vector kernel (x += alpha p, r -= alpha Ap, r.r): 1 (default) the block that finishes last
 *                     also forms beta, the stop flag and the iteration's record (4 launches per iteration); 2 every block also
 *                     forms alpha at its head (3 launches); 0 separate alpha and beta kernels (5 launches).  Same reduction
 *                     orders, same bits; 281-283 us per iteration at 256^3 in all three (the replayed graph hides the launches)
 *   "cg_pdl":         1: that kernel and the direction kernel are launched with programmatic stream serialization (default 0: no gain)
 *   "cg_fused_dot":   1 (default) spmvb_cg_solve takes p.Ap from the SpMV kernel when that kernel offers it (pattern format,
 *                     tensor ring, whole square grid): one pass over p and Ap less per iteration; 0 always runs the dot
 *   "last_cg_fused_dot": read-only, 1 when the last spmvb_cg_solve took p.Ap from the SpMV kernel
 *   "cg_keep_workspace": 1 (default) spmvb_cg_solve keeps its three work vectors (3n doubles) on the matrix handle
 *                     between solves, released by spmvb_matrix_destroy; 0 allocates and frees them in every solve
 *   "ell_kernel":     0 auto (one bulk-copied tile per CTA: 32 rows for ELL, 128 for vt), 2 tiles staged with vector loads,
 *                     3 the persistent two-stage TMA ring (ELL); 1 naive (ELL) and 3 for vt exist in lab builds only (the default
 *                     build runs its default kernel for them); lab build only: 4-7 other tile heights
 *   "box_prefetch", "box_prefetch_l1": L2 / L1 prefetch distance of the sliding-window kernels
 *   "debug_nochain":  lab build only, measurement only (1: sliding-window kernels skip their FP64 chains -- wrong results;
 *                     7: tensor ring without the per-plane-group line rotation -- same results)
 *   "last_pattern_kernel" (read): family of the last pattern launch: 1 List 1, 2 one-column box, 3 sliding window,
 *                     4 lab variant, 9 tensor ring */
int spmvb_set_option(const char *key, int value);
int spmvb_get_option(const char *key, int *value);

/* ---- upload: the reference structs' arrays, byte for byte ------------------- */
/* EllMatrix (inc/ell.hpp:14-24).  row_offset = global id of row 0 (0 for a whole matrix). */
int spmvb_ell_upload(int32_t n, int32_t width, int64_t nnz, int64_t row_offset, const double *values,
                     const int32_t *columns, spmvb_matrix **out);
/* VtCompressedMatrix (inc/compress.hpp:35-44). */
int spmvb_vt_upload(int32_t n, int32_t width, int32_t m, int64_t row_offset, const double *table,
                    const int32_t *sorted_columns, const int32_t *ends, spmvb_matrix **out);
/* PatternCompressedMatrix (inc/compress.hpp:52-76): patterns flattened as
 * disp_offsets[P+1] / disp_flat / ends_flat[P*m]; exception block may be empty
 * (n_exc = 0, pointers NULL).  Validates like validate() (inc/compress.hpp:95)
 * when check != 0 and n_cols > 0. */
int spmvb_pattern_upload(int32_t n, int32_t m, int64_t row_offset, const double *table,
                         int32_t n_patterns, const int64_t *disp_offsets, const int32_t *disp_flat,
                         const int32_t *ends_flat, const int32_t *row_pattern, int32_t values_in_pattern,
                         int32_t n_exc, int32_t w_exc, const int32_t *exc_rows, const double *exc_values,
                         const int32_t *exc_columns, spmvb_matrix **out);
/* StencilMatrix (inc/stencil.hpp:19-36, stencil_from_rows :47-50): validates
 * strictly ascending in-range columns. n_cols = global column count. */
int spmvb_csr_upload(int32_t n, int64_t n_cols, int64_t row_offset, const int64_t *row_start,
                     const int32_t *cols, const double *vals, spmvb_matrix **out);

/* ---- device-side build ------------------------------------------------------ */
/* generate_matrix (inc/stencil.hpp:40-45) for global rows [row_begin,row_end)
 * of the grid, as a device CSR handle (columns are global). */
int spmvb_generate_csr(const spmvb_grid *grid, int64_t row_begin, int64_t row_end, void *stream,
                       spmvb_matrix **out);
/* to_ell (inc/ell.hpp:28-29); min_width lets a slab use the global width. */
int spmvb_csr_to_ell(const spmvb_matrix *csr, int32_t min_width, void *stream, spmvb_matrix **out);
/* compress_values (inc/compress.hpp:82). */
int spmvb_csr_compress_values(const spmvb_matrix *csr, const spmvb_compress_options *opts,
                              int32_t min_width, void *stream, spmvb_matrix **out);
/* compress_patterns (inc/compress.hpp:84-85) + exception rows. */
int spmvb_csr_compress_patterns(const spmvb_matrix *csr, const spmvb_compress_options *opts,
                                void *stream, spmvb_matrix **out);
/* decompress / to_stencil (inc/compress.hpp:87-90, inc/ell.hpp:31-32): any
 * format back to a device CSR handle, columns re-sorted ascending. */
int spmvb_to_csr(const spmvb_matrix *a, void *stream, spmvb_matrix **out);
/* validate (inc/compress.hpp:92-95) on the device arrays; n_cols = global
 * column count.  SPMVB_ERR_INTEGRITY on any violation. */
int spmvb_validate(const spmvb_matrix *a, int64_t n_cols, void *stream);
/* Multi-slab dictionary merge: replace this handle's dictionary by `merged`
 * (same flattened layout as spmvb_pattern_upload) and remap row_pattern through
 * old_to_new[n_patterns_old]. */
int spmvb_pattern_remap(spmvb_matrix *a, int32_t n_patterns, const int64_t *disp_offsets,
                        const int32_t *disp_flat, const int32_t *ends_flat, const int32_t *old_to_new,
                        void *stream);

/* First local row of every pattern (n_patterns entries; -1 when unknown, e.g.
 * after upload).  With row_offset it gives the global first occurrence used to
 * merge per-slab dictionaries into the single-matrix numbering. */
int spmvb_pattern_first_rows(const spmvb_matrix *a, int32_t *out);

/* ---- introspection / download (bit-exact stream comparison) ------------------ */
int spmvb_matrix_get_info(const spmvb_matrix *a, spmvb_matrix_info *info);
int spmvb_matrix_stream_bytes(const spmvb_matrix *a, int32_t stream_id, uint64_t *bytes);
int spmvb_matrix_download(const spmvb_matrix *a, int32_t stream_id, uint64_t offset, uint64_t bytes,
                          void *dst);
/* raw device pointer of a stream (for torch / NCCL callers); NULL when absent */
int spmvb_matrix_stream_ptr(const spmvb_matrix *a, int32_t stream_id, void **dev_ptr);
int spmvb_matrix_destroy(spmvb_matrix *a);

/* ---- vectors (inc/stencil.hpp:14,54-59) ------------------------------------- */
int spmvb_vec_alloc(int64_t n, double **dev);
int spmvb_vec_free(double *dev);
int spmvb_vec_upload(double *dev, const double *host, int64_t n, void *stream);
int spmvb_vec_download(double *host, const double *dev, int64_t n, void *stream);
/* make_test_vector on the device: kind 0 ones, 1 linear, 2 random in [lo,hi);
 * element i is a pure function of (seed, first_index + i). */
int spmvb_vec_fill(double *dev, int64_t n, int32_t kind, uint64_t seed, double lo, double hi,
                   int64_t first_index, void *stream);

/* ---- SpMV (inc/kernels.hpp:19-36) -------------------------------------------- */
/* unchecked::spmv_rows: y[i] = (A x)[i] for local rows [row_begin,row_end),
 * overwrite, other rows untouched.  x_dev[j] holds the entry of global column
 * x_col0 + j, j in [0,x_len); a whole matrix uses x_col0 = 0, x_len = n; a
 * z-slab passes its ghosted local vector.  Asynchronous on `stream`. */
int spmvb_spmv(const spmvb_matrix *a, const double *x_dev, int64_t x_col0, int64_t x_len, double *y_dev,
               int32_t row_begin, int32_t row_end, void *stream);
/* spmv(fmt, Vector) -> Vector with HOST buffers (inc/kernels.hpp:23-25): checks
 * x_len == n (length mismatch -> SPMVB_ERR_INVALID_ARGUMENT), copies x to the
 * device, runs, copies y back, synchronises. */
int spmvb_spmv_host(const spmvb_matrix *a, const double *x_host, int64_t x_len, double *y_host);

/* ---- z-slab SpMV with halo exchange (SURVEY 8b "spmv_multi", 8e) ---------------- */
/* The grid is cut into z-slabs; a slab's rows are a contiguous range, exactly the [begin,end) of
 * unchecked::spmv_rows (inc/kernels.hpp:27-36; the paper's distribution: PAPER.md:473-477,505-531).  `a` holds the
 * rows of whole planes (plane_rows = nx*ny each; row_offset a multiple of it; global columns).  The slab's vector is
 *     x_ghosted = [ghost plane | owned planes | ghost plane],  n + 2*plane_rows entries,
 * i.e. spmvb_spmv's x_col0 = row_offset - plane_rows.  has_lower / has_upper: a neighbour exists on that side. */
typedef struct spmvb_slab spmvb_slab; /* opaque, caller-destroyed; not re-entrant */
enum spmvb_slab_mode {
    SPMVB_SLAB_SERIAL = 0, /* ghost copies, then one launch over all owned planes */
    SPMVB_SLAB_OVERLAP = 1 /* ghost copies on a side stream || planes that need no ghost; then the first and last plane */
};
int spmvb_slab_create(const spmvb_matrix *a, int64_t plane_rows, int32_t has_lower, int32_t has_upper, spmvb_slab **out);
int spmvb_slab_destroy(spmvb_slab *s);
/* One SpMV of the slab including its halo exchange as copies: lower_src = the lower neighbour's LAST owned plane,
 * upper_src = the upper neighbour's FIRST owned plane (device pointers: same device, peer-mapped, or from
 * spmvb_ipc_open; NULL = that ghost plane is already in place).  The neighbours' planes must not be written while the
 * call is in flight (the caller orders producers of x before it).  Asynchronous on `stream`.  From the second call
 * with the same pointers on, the copies and launches are replayed as one CUDA graph ("slab_graph" = 0: never). */
int spmvb_slab_spmv(spmvb_slab *s, double *x_ghosted, double *y, const double *lower_src, const double *upper_src,
                    int32_t mode, void *stream);
/* The two halves, for callers that run the exchange themselves (NCCL send/recv on their own stream): the rows that
 * need no ghost plane (may overlap the exchange), then the first and last owned planes (after the receive). */
int spmvb_slab_interior(spmvb_slab *s, const double *x_ghosted, double *y, void *stream);
int spmvb_slab_boundary(spmvb_slab *s, const double *x_ghosted, double *y, void *stream);
int spmvb_slab_last_was_graph(const spmvb_slab *s, int32_t *flag);
/* Peer memory across processes (one process per GPU): CUDA IPC handle of a vector from spmvb_vec_alloc. */
int spmvb_ipc_export(const void *dev_base, unsigned char handle[64]);
int spmvb_ipc_open(const unsigned char handle[64], void **dev_ptr);
int spmvb_ipc_close(void *dev_ptr);

/* One host thread driving G slabs over a device list (context over a device list, spmv_multi, bench).
 * Devices may repeat (logical slabs on one device).  Build is per slab on its device (generator -> format), the
 * per-slab pattern dictionaries are merged so that ids equal a single-matrix compression; slab g owns planes
 * [z0,z1) of grid->nz split as evenly as possible (low slabs take the remainder). */
typedef struct spmvb_multi spmvb_multi;
int spmvb_multi_create(const spmvb_grid *grid, int32_t format, const spmvb_compress_options *opts, const int32_t *devices,
                       int32_t n_devices, spmvb_multi **out);
int spmvb_multi_destroy(spmvb_multi *m);
int spmvb_multi_parts(const spmvb_multi *m, int32_t *n_parts);
/* any out pointer may be NULL */
int spmvb_multi_part(const spmvb_multi *m, int32_t part, int32_t *device, int64_t *z0, int64_t *z1,
                     const spmvb_matrix **matrix, double **x_ghosted, double **y);
int spmvb_multi_fill_x(spmvb_multi *m, int32_t kind, uint64_t seed, double lo, double hi); /* make_test_vector, global */
int spmvb_multi_upload_x(spmvb_multi *m, const double *x_host, int64_t n);
int spmvb_multi_download_y(spmvb_multi *m, double *y_host, int64_t n);
int spmvb_multi_spmv(spmvb_multi *m, int32_t mode); /* y = A x on every slab, exchange included; asynchronous */
int spmvb_multi_sync(spmvb_multi *m);
/* reps SpMVs after a warm-up: host wall clock between device-wide syncs and the slowest slab's device time */
int spmvb_multi_bench(spmvb_multi *m, int32_t reps, int32_t mode, double *seconds, double *device_seconds);

/* ---- the caller of the path: CG vector primitives and driver ---- */
/* dot (inc/kernels.hpp:39): device vectors, result to the host; fixed-shape tree (deterministic). */
int spmvb_dot(const double *u_dev, const double *v_dev, int64_t n, double *result, void *stream);
/* waxpby_into (inc/kernels.hpp:41-42): w = alpha*x + beta*y, bit-identical to the reference expression;
 * w may alias x or y. */
int spmvb_waxpby(double alpha, const double *x_dev, double beta, const double *y_dev, double *w_dev, int64_t n,
                 void *stream);
/* cg_solve (inc/solver.hpp:40-46) without preconditioner, x0 = 0, SpMV on the handle's format:
 * per iteration 1 SpMV, 3 dots, 3 waxpbys.  residual_history (may be NULL) needs max_iterations+1
 * slots: [0] = 1.0, [k] = ||r_k|| / ||b||.  SPMVB_ERR_DIVERGENCE on a non-finite value
 * (iteration in the message and in *iterations). */
int spmvb_cg_solve(const spmvb_matrix *a, const double *b_dev, double *x_dev, int32_t max_iterations, double tolerance,
                   int32_t *iterations, int32_t *converged, double *residual_history, void *stream);

/* symgs_sweep (inc/kernels.hpp:44-48): one forward then one backward Gauss-Seidel sweep in natural
 * order, in place, on the whole square matrix as a CSR handle whose rows are the nodes of `grid` (only nx, ny, nz are
 * read).  Bit-identical to the sequential loop: the rows are processed by hyperplanes ix + 2 iy + 4 iz, which order every
 * coupling of a 27-point (or sparser) stencil the way the row index does; the schedule is verified against the matrix
 * first.  SPMVB_ERR_INVALID_ARGUMENT for a zero or missing diagonal (the reference's singularity error) and for a matrix
 * with couplings the schedule does not order (nothing is written in either case). */
int spmvb_symgs_sweep(const spmvb_matrix *csr, const spmvb_grid *grid, double *x_dev, const double *b_dev, void *stream);
/* cg_solve (inc/solver.hpp:40-46) with the SymGS preconditioner: z = symgs_sweeps sweeps on A z = r from a zero guess
 * (SPEC.md:311,327); `a` is the SpMV backend (any format), `csr` the same matrix for the sweeps.  Per iteration 1 SpMV,
 * 3 dots (p.Ap, r.r, r.z), 3 waxpbys, 1 preconditioner application.  History and errors as spmvb_cg_solve. */
int spmvb_pcg_solve(const spmvb_matrix *a, const spmvb_matrix *csr, const spmvb_grid *grid, int32_t symgs_sweeps, const double *b_dev,
                    double *x_dev, int32_t max_iterations, double tolerance, int32_t *iterations, int32_t *converged,
                    double *residual_history, void *stream);

/* ---- verification helpers ----------------------------------------------------- */
/* max_i |y[i]-ref[i]| / den[i] and the number of entries whose bit patterns
 * differ.  den = scale[i] (= sum_k |a_ik x_k|, from spmvb_row_abs_scale) when a
 * scale is given -- the per-row measure used between formats whose summation
 * orders differ -- else |ref[i]| (1 where that is 0).  Device pointers. */
int spmvb_compare(const double *y, const double *ref, const double *scale, int64_t n, double *max_rel,
                  int64_t *n_bit_mismatch, void *stream);
/* sum_k |a_ik x_k| per local row (CSR handle), the scale above. */
int spmvb_row_abs_scale(const spmvb_matrix *csr, const double *x_dev, int64_t x_col0, double *scale_dev,
                        void *stream);

#ifdef __cplusplus
}
#endif
#endif
