"""ctypes binding of libspmvcomp_b200.so (the C-ABI in include/spmvcomp_b200.h).

There is no CPU fallback: if the CUDA library is missing this module raises at
import, and every compute call fails with CudaError when no device is present.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("SPMVB_LIB") or os.path.join(_HERE, "libspmvcomp_b200.so")  # SPMVB_LIB: another build of the same C-ABI (e.g. the lab build)


class SpmvcompError(RuntimeError):
    code = -1


class InvalidArgument(SpmvcompError, ValueError):  # std::invalid_argument (grid.hpp:35-47)
    code = 1


class TableOverflowError(SpmvcompError):  # errors.hpp:9
    code = 2


class IntegrityError(SpmvcompError):  # errors.hpp:16
    code = 3


class VerificationError(SpmvcompError):  # errors.hpp:33
    code = 4


class IoError(SpmvcompError):  # errors.hpp:39
    code = 5


class DivergenceError(SpmvcompError):  # errors.hpp:22
    code = 6


class CudaError(SpmvcompError):
    code = 7


class NcclError(SpmvcompError):
    code = 8


class OutOfMemory(SpmvcompError, MemoryError):
    code = 9


_ERRORS = {c.code: c for c in (InvalidArgument, TableOverflowError, IntegrityError, VerificationError, IoError,
                               DivergenceError, CudaError, NcclError, OutOfMemory)}

FMT_ELL, FMT_VT, FMT_PATTERN, FMT_CSR = 0, 1, 2, 3
(S_VALUES, S_COLUMNS, S_TABLE, S_SORTED_COLUMNS, S_ENDS, S_ROW_PATTERN, S_DISP_OFFSETS, S_DISP_FLAT, S_ENDS_FLAT,
 S_EXC_ROWS, S_EXC_VALUES, S_EXC_COLUMNS, S_CSR_ROW_START, S_CSR_COLS, S_CSR_VALS) = range(15)


class MatrixInfo(C.Structure):
    _fields_ = [("format", C.c_int32), ("n", C.c_int32), ("width", C.c_int32), ("m", C.c_int32),
                ("n_patterns", C.c_int32), ("n_exc", C.c_int32), ("w_exc", C.c_int32),
                ("values_in_pattern", C.c_int32), ("nnz", C.c_int64), ("row_offset", C.c_int64),
                ("disp_total", C.c_int64), ("device", C.c_int32), ("kernel_plan", C.c_int32),
                ("box_stride_y", C.c_int32), ("box_stride_z", C.c_int32), ("reserved_", C.c_int32)]


class Grid(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("diagonal", C.c_double),
                ("off_diagonal", C.c_double), ("perturb", C.c_int32), ("perturb_seed", C.c_uint64),
                ("perturb_fraction", C.c_double), ("perturb_noise", C.c_double)]


class CompressOptions(C.Structure):
    _fields_ = [("value_table_limit", C.c_uint64), ("values_in_pattern", C.c_int32),
                ("min_pattern_rows", C.c_int32), ("dict_cap", C.c_int32)]


# every symbol include/spmvcomp_b200.h declares (tests check the library exports all of them)
SYMBOLS = [
    "spmvb_last_error", "spmvb_version", "spmvb_device_count", "spmvb_set_device", "spmvb_set_option",
    "spmvb_get_option", "spmvb_ell_upload", "spmvb_vt_upload", "spmvb_pattern_upload", "spmvb_csr_upload",
    "spmvb_generate_csr", "spmvb_csr_to_ell", "spmvb_csr_compress_values", "spmvb_csr_compress_patterns",
    "spmvb_to_csr", "spmvb_validate", "spmvb_pattern_remap", "spmvb_pattern_first_rows", "spmvb_matrix_get_info",
    "spmvb_matrix_stream_bytes", "spmvb_matrix_download", "spmvb_matrix_stream_ptr", "spmvb_matrix_destroy",
    "spmvb_vec_alloc", "spmvb_vec_free", "spmvb_vec_upload", "spmvb_vec_download", "spmvb_vec_fill",
    "spmvb_spmv", "spmvb_spmv_host", "spmvb_compare", "spmvb_row_abs_scale", "spmvb_dot", "spmvb_waxpby",
    "spmvb_cg_solve", "spmvb_symgs_sweep", "spmvb_pcg_solve",
    "spmvb_slab_create", "spmvb_slab_destroy", "spmvb_slab_spmv", "spmvb_slab_interior", "spmvb_slab_boundary",
    "spmvb_slab_last_was_graph", "spmvb_ipc_export", "spmvb_ipc_open", "spmvb_ipc_close",
    "spmvb_multi_create", "spmvb_multi_destroy", "spmvb_multi_parts", "spmvb_multi_part", "spmvb_multi_fill_x",
    "spmvb_multi_upload_x", "spmvb_multi_download_y", "spmvb_multi_spmv", "spmvb_multi_sync", "spmvb_multi_bench",
]
SLAB_SERIAL, SLAB_OVERLAP = 0, 1

if not os.path.exists(SO_PATH):
    raise ImportError(
        f"{SO_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(nvcc, sm_100a). There is no CPU fallback.")

lib = C.CDLL(SO_PATH)
lib.spmvb_last_error.restype = C.c_char_p
_vp, _i32, _i64, _u64, _f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
_pp = C.POINTER(C.c_void_p)
lib.spmvb_ell_upload.argtypes = [_i32, _i32, _i64, _i64, _vp, _vp, _pp]
lib.spmvb_vt_upload.argtypes = [_i32, _i32, _i32, _i64, _vp, _vp, _vp, _pp]
lib.spmvb_pattern_upload.argtypes = [_i32, _i32, _i64, _vp, _i32, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp,
                                     _vp, _pp]
lib.spmvb_csr_upload.argtypes = [_i32, _i64, _i64, _vp, _vp, _vp, _pp]
lib.spmvb_generate_csr.argtypes = [C.POINTER(Grid), _i64, _i64, _vp, _pp]
lib.spmvb_csr_to_ell.argtypes = [_vp, _i32, _vp, _pp]
lib.spmvb_csr_compress_values.argtypes = [_vp, C.POINTER(CompressOptions), _i32, _vp, _pp]
lib.spmvb_csr_compress_patterns.argtypes = [_vp, C.POINTER(CompressOptions), _vp, _pp]
lib.spmvb_to_csr.argtypes = [_vp, _vp, _pp]
lib.spmvb_validate.argtypes = [_vp, _i64, _vp]
lib.spmvb_pattern_remap.argtypes = [_vp, _i32, _vp, _vp, _vp, _vp, _vp]
lib.spmvb_pattern_first_rows.argtypes = [_vp, _vp]
lib.spmvb_matrix_get_info.argtypes = [_vp, C.POINTER(MatrixInfo)]
lib.spmvb_matrix_stream_bytes.argtypes = [_vp, _i32, C.POINTER(_u64)]
lib.spmvb_matrix_download.argtypes = [_vp, _i32, _u64, _u64, _vp]
lib.spmvb_matrix_stream_ptr.argtypes = [_vp, _i32, _pp]
lib.spmvb_matrix_destroy.argtypes = [_vp]
lib.spmvb_vec_alloc.argtypes = [_i64, _pp]
lib.spmvb_vec_free.argtypes = [_vp]
lib.spmvb_vec_upload.argtypes = [_vp, _vp, _i64, _vp]
lib.spmvb_vec_download.argtypes = [_vp, _vp, _i64, _vp]
lib.spmvb_vec_fill.argtypes = [_vp, _i64, _i32, _u64, _f64, _f64, _i64, _vp]
lib.spmvb_spmv.argtypes = [_vp, _vp, _i64, _i64, _vp, _i32, _i32, _vp]
lib.spmvb_spmv_host.argtypes = [_vp, _vp, _i64, _vp]
lib.spmvb_compare.argtypes = [_vp, _vp, _vp, _i64, C.POINTER(_f64), C.POINTER(_i64), _vp]
lib.spmvb_row_abs_scale.argtypes = [_vp, _vp, _i64, _vp, _vp]
lib.spmvb_dot.argtypes = [_vp, _vp, _i64, C.POINTER(_f64), _vp]
lib.spmvb_waxpby.argtypes = [_f64, _vp, _f64, _vp, _vp, _i64, _vp]
lib.spmvb_cg_solve.argtypes = [_vp, _vp, _vp, _i32, _f64, C.POINTER(_i32), C.POINTER(_i32), _vp, _vp]
lib.spmvb_symgs_sweep.argtypes = [_vp, C.POINTER(Grid), _vp, _vp, _vp]
lib.spmvb_pcg_solve.argtypes = [_vp, _vp, C.POINTER(Grid), _i32, _vp, _vp, _i32, _f64, C.POINTER(_i32), C.POINTER(_i32), _vp, _vp]
lib.spmvb_slab_create.argtypes = [_vp, _i64, _i32, _i32, _pp]
lib.spmvb_slab_destroy.argtypes = [_vp]
lib.spmvb_slab_spmv.argtypes = [_vp, _vp, _vp, _vp, _vp, _i32, _vp]
lib.spmvb_slab_interior.argtypes = [_vp, _vp, _vp, _vp]
lib.spmvb_slab_boundary.argtypes = [_vp, _vp, _vp, _vp]
lib.spmvb_slab_last_was_graph.argtypes = [_vp, C.POINTER(_i32)]
lib.spmvb_ipc_export.argtypes = [_vp, C.c_char_p]
lib.spmvb_ipc_open.argtypes = [C.c_char_p, _pp]
lib.spmvb_ipc_close.argtypes = [_vp]
lib.spmvb_multi_create.argtypes = [C.POINTER(Grid), _i32, C.POINTER(CompressOptions), C.POINTER(_i32), _i32, _pp]
lib.spmvb_multi_destroy.argtypes = [_vp]
lib.spmvb_multi_parts.argtypes = [_vp, C.POINTER(_i32)]
lib.spmvb_multi_part.argtypes = [_vp, _i32, C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_i64), _pp, _pp, _pp]
lib.spmvb_multi_fill_x.argtypes = [_vp, _i32, _u64, _f64, _f64]
lib.spmvb_multi_upload_x.argtypes = [_vp, _vp, _i64]
lib.spmvb_multi_download_y.argtypes = [_vp, _vp, _i64]
lib.spmvb_multi_spmv.argtypes = [_vp, _i32]
lib.spmvb_multi_sync.argtypes = [_vp]
lib.spmvb_multi_bench.argtypes = [_vp, _i32, _i32, C.POINTER(_f64), C.POINTER(_f64)]
lib.spmvb_set_option.argtypes = [C.c_char_p, C.c_int]
lib.spmvb_get_option.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
lib.spmvb_device_count.argtypes = [C.POINTER(C.c_int)]


def check(rc):
    if rc != 0:
        raise _ERRORS.get(rc, SpmvcompError)(lib.spmvb_last_error().decode())
