"""Host-side mirror of the reference's C++ interface for the SpMV path, as thin
wrappers over the C-ABI (include/spmvcomp_b200.h).  Names, argument meaning and
error behaviour follow /root/reference/proj/include/spmvcomp (cited per symbol);
all computation happens on the GPU -- there is no CPU path in this package.

Matrices are device-resident handles (`DeviceMatrix`); vectors are device arrays
(`DeviceVector`, or anything with a `.data_ptr()` such as a CUDA torch tensor).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _cabi as cabi
from ._cabi import (FMT_CSR, FMT_ELL, FMT_PATTERN, FMT_VT, CudaError, IntegrityError, InvalidArgument,  # noqa: F401
                    SpmvcompError, TableOverflowError, VerificationError, check, lib)

K_MAX_ROWS = (1 << 31) - 1  # grid.hpp:11 kMaxRows
ONES, LINEAR, RANDOM = 0, 1, 2  # stencil.hpp:54 VectorKind

_DTYPES = {
    cabi.S_VALUES: np.float64, cabi.S_COLUMNS: np.int32, cabi.S_TABLE: np.float64,
    cabi.S_SORTED_COLUMNS: np.int32, cabi.S_ENDS: np.int32, cabi.S_ROW_PATTERN: np.int32,
    cabi.S_DISP_OFFSETS: np.int64, cabi.S_DISP_FLAT: np.int32, cabi.S_ENDS_FLAT: np.int32,
    cabi.S_EXC_ROWS: np.int32, cabi.S_EXC_VALUES: np.float64, cabi.S_EXC_COLUMNS: np.int32,
    cabi.S_CSR_ROW_START: np.int64, cabi.S_CSR_COLS: np.int32, cabi.S_CSR_VALS: np.float64,
}
_NAMES = {
    "values": cabi.S_VALUES, "columns": cabi.S_COLUMNS, "table": cabi.S_TABLE,
    "sorted_columns": cabi.S_SORTED_COLUMNS, "ends": cabi.S_ENDS, "row_pattern": cabi.S_ROW_PATTERN,
    "disp_offsets": cabi.S_DISP_OFFSETS, "disp_flat": cabi.S_DISP_FLAT, "ends_flat": cabi.S_ENDS_FLAT,
    "exc_rows": cabi.S_EXC_ROWS, "exc_values": cabi.S_EXC_VALUES, "exc_columns": cabi.S_EXC_COLUMNS,
    "row_start": cabi.S_CSR_ROW_START, "cols": cabi.S_CSR_COLS, "vals": cabi.S_CSR_VALS,
}


@dataclass(frozen=True)
class GridSpec:
    """grid.hpp:15-33."""
    nx: int = 1
    ny: int = 1
    nz: int = 1

    def rows(self) -> int:
        return self.nx * self.ny * self.nz

    def node(self, ix, iy, iz) -> int:
        return ix + self.nx * (iy + self.ny * iz)


def validate_grid(g: GridSpec):
    """grid.hpp:35-47."""
    if g.nx < 1 or g.ny < 1 or g.nz < 1:
        raise InvalidArgument(f"grid dimensions must be >= 1, got {g.nx}x{g.ny}x{g.nz}")
    if g.rows() > K_MAX_ROWS:
        raise InvalidArgument(f"grid {g.nx}x{g.ny}x{g.nz} has {g.rows()} rows; column indices must fit a "
                              "4-byte signed integer")


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    if isinstance(a, DeviceVector):
        return C.c_void_p(a.ptr)
    return a.ctypes.data_as(C.c_void_p)


def _stream(stream):
    if stream is None:
        return None
    return C.c_void_p(getattr(stream, "cuda_stream", stream))


def _np(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class DeviceVector:
    """A length-n fp64 device array (Vector, stencil.hpp:14)."""

    def __init__(self, n: int):
        p = C.c_void_p()
        check(lib.spmvb_vec_alloc(n, C.byref(p)))
        self.ptr, self.n = p.value, n

    def __del__(self):
        if getattr(self, "ptr", None):
            lib.spmvb_vec_free(C.c_void_p(self.ptr))
            self.ptr = None

    def data_ptr(self):
        return self.ptr

    @property
    def __cuda_array_interface__(self):
        """Zero-copy view for torch.as_tensor(v, device="cuda") and friends (the vector stays owned by this object)."""
        return {"shape": (self.n,), "typestr": "<f8", "data": (self.ptr, False), "version": 2}

    @classmethod
    def from_host(cls, host, stream=None):
        host = _np(host, np.float64)
        v = cls(host.shape[0])
        check(lib.spmvb_vec_upload(C.c_void_p(v.ptr), _ptr(host), host.shape[0], _stream(stream)))
        return v

    def to_host(self, stream=None):
        out = np.empty(self.n, dtype=np.float64)
        check(lib.spmvb_vec_download(_ptr(out), C.c_void_p(self.ptr), self.n, _stream(stream)))
        return out

    def fill(self, kind, seed=None, lo=0.0, hi=1.0, first_index=0, stream=None):
        if kind == RANDOM and seed is None:
            raise InvalidArgument("seed is required for the random kind")  # stencil.hpp:56-57
        check(lib.spmvb_vec_fill(C.c_void_p(self.ptr), self.n, kind, seed or 0, lo, hi, first_index, _stream(stream)))
        return self


def make_test_vector(n, kind, seed=None, lo=0.0, hi=1.0, first_index=0, stream=None) -> DeviceVector:
    """make_test_vector (stencil.hpp:54-59) on the device; [lo,hi) defaults to the header's [0,1)."""
    if n < 1:
        raise InvalidArgument("vector length must be >= 1")
    return DeviceVector(n).fill(kind, seed, lo, hi, first_index, stream)


class DeviceMatrix:
    """Opaque device-resident matrix in one of the reference's formats."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            lib.spmvb_matrix_destroy(self.h)
            self.h = None

    @property
    def info(self) -> cabi.MatrixInfo:
        i = cabi.MatrixInfo()
        check(lib.spmvb_matrix_get_info(self.h, C.byref(i)))
        return i

    n = property(lambda self: self.info.n)
    nnz = property(lambda self: self.info.nnz)
    format = property(lambda self: self.info.format)

    def stream_bytes(self, name) -> int:
        b = C.c_uint64()
        check(lib.spmvb_matrix_stream_bytes(self.h, _NAMES[name], C.byref(b)))
        return b.value

    def download(self, name, offset_elems=0, count=None) -> np.ndarray:
        """Copy one device stream back (bit-exact comparison against the oracle)."""
        sid = _NAMES[name]
        dt = np.dtype(_DTYPES[sid])
        total = self.stream_bytes(name) // dt.itemsize
        count = total - offset_elems if count is None else count
        out = np.empty(count, dtype=dt)
        check(lib.spmvb_matrix_download(self.h, sid, offset_elems * dt.itemsize, count * dt.itemsize, _ptr(out)))
        return out

    def stream_ptr(self, name) -> int:
        p = C.c_void_p()
        check(lib.spmvb_matrix_stream_ptr(self.h, _NAMES[name], C.byref(p)))
        return p.value or 0


def _wrap(call, *args):
    out = C.c_void_p()
    check(call(*args, C.byref(out)))
    return DeviceMatrix(out)


# ---- upload of the reference structs' arrays --------------------------------------
def upload_ell(n, width, nnz, values, columns, row_offset=0) -> DeviceMatrix:
    """EllMatrix (ell.hpp:14-24)."""
    values, columns = _np(values, np.float64), _np(columns, np.int32)
    if values.size != n * width or columns.size != n * width:
        raise InvalidArgument("EllMatrix arrays must hold n*width entries")
    return _wrap(lib.spmvb_ell_upload, n, width, nnz, row_offset, _ptr(values), _ptr(columns))


def upload_vt(n, width, table, sorted_columns, ends, row_offset=0) -> DeviceMatrix:
    """VtCompressedMatrix (compress.hpp:35-44)."""
    table, sc, ends = _np(table, np.float64), _np(sorted_columns, np.int32), _np(ends, np.int32)
    m = table.size
    if sc.size != n * width or ends.size != n * m:
        raise InvalidArgument("VtCompressedMatrix arrays have the wrong size")
    return _wrap(lib.spmvb_vt_upload, n, width, m, row_offset, _ptr(table), _ptr(sc), _ptr(ends))


def upload_pattern(n, table, disp_offsets, disp_flat, ends_flat, row_pattern, values_in_pattern=False,
                   exc_rows=None, exc_values=None, exc_columns=None, w_exc=0, row_offset=0) -> DeviceMatrix:
    """PatternCompressedMatrix (compress.hpp:52-76) with the optional exception block."""
    table = _np(table, np.float64)
    do, df, ef = _np(disp_offsets, np.int64), _np(disp_flat, np.int32), _np(ends_flat, np.int32)
    rp = _np(row_pattern, np.int32)
    n_pat = do.size - 1
    if rp.size != n or ef.size != n_pat * table.size or df.size != (do[-1] if do.size else 0):
        raise InvalidArgument("PatternCompressedMatrix arrays have the wrong size")
    er = _np(exc_rows if exc_rows is not None else [], np.int32)
    ev = _np(exc_values if exc_values is not None else [], np.float64)
    ec = _np(exc_columns if exc_columns is not None else [], np.int32)
    return _wrap(lib.spmvb_pattern_upload, n, table.size, row_offset, _ptr(table), n_pat, _ptr(do), _ptr(df),
                 _ptr(ef), _ptr(rp), int(values_in_pattern), er.size, w_exc, _ptr(er), _ptr(ev), _ptr(ec))


def upload_csr(n, row_start, cols, vals, n_cols=None, row_offset=0) -> DeviceMatrix:
    """StencilMatrix / stencil_from_rows (stencil.hpp:19-36,47-50)."""
    rs, cols, vals = _np(row_start, np.int64), _np(cols, np.int32), _np(vals, np.float64)
    return _wrap(lib.spmvb_csr_upload, n, n if n_cols is None else n_cols, row_offset, _ptr(rs), _ptr(cols),
                 _ptr(vals))


def stencil_from_rows(n, rows) -> DeviceMatrix:
    """stencil_from_rows (stencil.hpp:47-50): rows = per-row lists of (column, value)."""
    rs = np.zeros(n + 1, dtype=np.int64)
    cols, vals = [], []
    for i, r in enumerate(rows):
        rs[i + 1] = rs[i] + len(r)
        cols += [c for c, _ in r]
        vals += [v for _, v in r]
    return upload_csr(n, rs, cols, vals)


# ---- device-side build --------------------------------------------------------------
def generate_matrix(spec: GridSpec, diagonal=26.0, off_diagonal=-1.0, perturb=None, row_begin=0, row_end=None,
                    stream=None) -> DeviceMatrix:
    """generate_matrix (stencil.hpp:40-45) on the device, as a CSR handle.  `perturb`
    = (seed, fraction, noise) enables BASELINE.json's config-4 recipe; [row_begin,row_end)
    selects a slab of global rows."""
    validate_grid(spec)
    g = cabi.Grid(spec.nx, spec.ny, spec.nz, diagonal, off_diagonal, 0, 0, 0.0, 0.0)
    if perturb is not None:
        g.perturb, g.perturb_seed, g.perturb_fraction, g.perturb_noise = 1, perturb[0], perturb[1], perturb[2]
    row_end = spec.rows() if row_end is None else row_end
    return _wrap(lib.spmvb_generate_csr, C.byref(g), row_begin, row_end, _stream(stream))


def to_ell(m: DeviceMatrix, min_width=0, stream=None) -> DeviceMatrix:
    """to_ell (ell.hpp:28-29)."""
    return _wrap(lib.spmvb_csr_to_ell, m.h, min_width, _stream(stream))


def _opts(limit, values_in_pattern=False, min_pattern_rows=1, dict_cap=0):
    return cabi.CompressOptions(limit, int(values_in_pattern), min_pattern_rows, dict_cap)


def compress_values(m: DeviceMatrix, value_table_limit=256, min_width=0, stream=None) -> DeviceMatrix:
    """compress_values (compress.hpp:82)."""
    return _wrap(lib.spmvb_csr_compress_values, m.h, C.byref(_opts(value_table_limit)), min_width, _stream(stream))


def compress_patterns(m: DeviceMatrix, values_in_pattern=False, value_table_limit=256, min_pattern_rows=1,
                      dict_cap=0, stream=None) -> DeviceMatrix:
    """compress_patterns (compress.hpp:84-85); min_pattern_rows >= 2 enables exception rows."""
    o = _opts(value_table_limit, values_in_pattern, min_pattern_rows, dict_cap)
    return _wrap(lib.spmvb_csr_compress_patterns, m.h, C.byref(o), _stream(stream))


def decompress(c: DeviceMatrix, stream=None) -> DeviceMatrix:
    """decompress / to_stencil (compress.hpp:87-90, ell.hpp:31-32) -> CSR handle."""
    return _wrap(lib.spmvb_to_csr, c.h, _stream(stream))


to_stencil = decompress


def pattern_first_rows(c: DeviceMatrix) -> np.ndarray:
    """First local row of each pattern of a device-built pattern handle (-1 = unknown)."""
    out = np.empty(c.info.n_patterns, dtype=np.int32)
    check(lib.spmvb_pattern_first_rows(c.h, _ptr(out)))
    return out


def pattern_remap(c: DeviceMatrix, disp_offsets, disp_flat, ends_flat, old_to_new, stream=None):
    """Install a merged dictionary and renumber row_pattern (multi-slab build)."""
    do, df = _np(disp_offsets, np.int64), _np(disp_flat, np.int32)
    ef, o2n = _np(ends_flat, np.int32), _np(old_to_new, np.int32)
    check(lib.spmvb_pattern_remap(c.h, do.size - 1, _ptr(do), _ptr(df), _ptr(ef), _ptr(o2n), _stream(stream)))


def validate(c: DeviceMatrix, n_cols=None, stream=None):
    """validate (compress.hpp:92-95)."""
    check(lib.spmvb_validate(c.h, c.n if n_cols is None else n_cols, _stream(stream)))


# ---- SpMV (kernels.hpp:19-36) -----------------------------------------------------------
def spmv_flops(nnz):
    return 2 * nnz  # kernels.hpp:14


def spmv_rows(a: DeviceMatrix, x, y, begin, end, x_col0=0, x_len=None, stream=None):
    """unchecked::spmv_rows (kernels.hpp:27-36): device x and y, rows [begin,end), asynchronous."""
    if x_len is None:
        x_len = x.n if isinstance(x, DeviceVector) else x.numel()
    check(lib.spmvb_spmv(a.h, _ptr(x), x_col0, x_len, _ptr(y), begin, end, _stream(stream)))


def spmv(a: DeviceMatrix, x) -> np.ndarray:
    """spmv (kernels.hpp:23-25) with host vectors: validated, returns a fresh vector.  The device arrays of a handle
    are immutable, so the structural validation (spmvb_validate: column / id ranges, group ends) runs once per handle."""
    x = _np(x, np.float64)
    if not getattr(a, "_validated", False):
        info = a.info
        if info.format in (FMT_ELL, FMT_VT, FMT_PATTERN) and info.row_offset == 0 and x.shape[0] == info.n:
            check(lib.spmvb_validate(a.h, info.n, None))  # whole square matrix: columns in [0, n)
            a._validated = True
    y = np.empty(a.n, dtype=np.float64)
    check(lib.spmvb_spmv_host(a.h, _ptr(x), x.shape[0], _ptr(y)))
    return y


def dot(u, v, n=None, stream=None) -> float:
    """dot (kernels.hpp:39) on device vectors."""
    n = u.n if n is None else n
    out = C.c_double()
    check(lib.spmvb_dot(_ptr(u), _ptr(v), n, C.byref(out), _stream(stream)))
    return out.value


def waxpby_into(alpha, x, beta, y, w, n=None, stream=None):
    """waxpby_into (kernels.hpp:42): w = alpha*x + beta*y on device vectors (w may alias x or y)."""
    n = x.n if n is None else n
    check(lib.spmvb_waxpby(alpha, _ptr(x), beta, _ptr(y), _ptr(w), n, _stream(stream)))


@dataclass
class CgReport:
    """solver.hpp:30-38 (flops per SPEC.md:321: 2*nnz + 6n + 6n per iteration, no preconditioner)."""
    iterations: int
    converged: bool
    residual_history: list
    flops_total: int

    def final_residual(self):
        return self.residual_history[-1]


def symgs_sweep(csr: DeviceMatrix, grid: GridSpec, x, b, stream=None):
    """symgs_sweep (kernels.hpp:44-48) in place on device vectors: the natural-order sweep by hyperplanes of `grid`."""
    g = cabi.Grid(grid.nx, grid.ny, grid.nz, 0.0, 0.0, 0, 0, 0.0, 0.0)
    check(lib.spmvb_symgs_sweep(csr.h, C.byref(g), _ptr(x), _ptr(b), _stream(stream)))


def cg_solve(a: DeviceMatrix, b, max_iterations=500, tolerance=1e-8, stream=None, symgs_sweeps=0, csr=None, grid=None, x=None):
    """cg_solve (solver.hpp:40-46) on the device.  b: device vector; returns (x, CgReport).  symgs_sweeps >= 1 preconditions
    with that many SymGS sweeps from a zero guess (needs the matrix as `csr` and its `grid`).  `x`: a device vector to
    receive the solution (repeated solves then allocate nothing: cudaMalloc / cudaFree of large vectors stall now and then)."""
    n = a.n
    x = DeviceVector(n) if x is None else x
    hist = np.zeros(max_iterations + 1, dtype=np.float64)
    it, conv = C.c_int32(), C.c_int32()
    if symgs_sweeps:
        if csr is None or grid is None:
            raise InvalidArgument("cg_solve: the SymGS preconditioner needs csr= and grid=")
        g = cabi.Grid(grid.nx, grid.ny, grid.nz, 0.0, 0.0, 0, 0, 0.0, 0.0)
        check(lib.spmvb_pcg_solve(a.h, csr.h, C.byref(g), symgs_sweeps, _ptr(b), _ptr(x), max_iterations, tolerance, C.byref(it),
                                  C.byref(conv), _ptr(hist), _stream(stream)))
        k = it.value
        applications = k + (0 if conv.value else 1)
        return x, CgReport(k, bool(conv.value), hist[:k + 1].tolist(), k * (2 * a.nnz + 12 * n) + applications * symgs_sweeps * 4 * a.nnz)
    check(lib.spmvb_cg_solve(a.h, _ptr(b), _ptr(x), max_iterations, tolerance, C.byref(it), C.byref(conv), _ptr(hist),
                             _stream(stream)))
    k = it.value
    return x, CgReport(k, bool(conv.value), hist[:k + 1].tolist(), k * (2 * a.nnz + 12 * n))


def compare(y, ref, n, scale=None, stream=None):
    """Device-side (max relative deviation, number of bit-different entries)."""
    worst, bad = C.c_double(), C.c_int64()
    check(lib.spmvb_compare(_ptr(y), _ptr(ref), _ptr(scale), n, C.byref(worst), C.byref(bad), _stream(stream)))
    return worst.value, bad.value


def row_abs_scale(csr: DeviceMatrix, x, out, x_col0=0, stream=None):
    check(lib.spmvb_row_abs_scale(csr.h, _ptr(x), x_col0, _ptr(out), _stream(stream)))


def set_option(key: str, value: int):
    check(lib.spmvb_set_option(key.encode(), value))


def get_option(key: str) -> int:
    v = C.c_int()
    check(lib.spmvb_get_option(key.encode(), C.byref(v)))
    return v.value


def device_count() -> int:
    c = C.c_int()
    check(lib.spmvb_device_count(C.byref(c)))
    return c.value


# ---- z-slabs behind the C-ABI (SURVEY 8b "spmv_multi", 8e) -----------------------------------------------------------
SLAB_SERIAL, SLAB_OVERLAP = cabi.SLAB_SERIAL, cabi.SLAB_OVERLAP


class Slab:
    """One rank's slab of whole planes: spmvb_slab_* (the row ranges of unchecked::spmv_rows, kernels.hpp:27-36).
    x is the ghosted local vector [ghost plane | owned planes | ghost plane]."""

    def __init__(self, a: DeviceMatrix, plane_rows: int, has_lower: bool, has_upper: bool):
        h = C.c_void_p()
        check(lib.spmvb_slab_create(a.h, plane_rows, int(has_lower), int(has_upper), C.byref(h)))
        self.h, self.a = h, a  # keeps the matrix alive

    def __del__(self):
        if getattr(self, "h", None):
            lib.spmvb_slab_destroy(self.h)
            self.h = None

    def spmv(self, x_ghosted, y, lower_src=None, upper_src=None, mode=SLAB_SERIAL, stream=None):
        """Exchange (copies from the neighbours' planes: device pointers or None) + SpMV; a CUDA graph from the second call on."""
        lo = None if lower_src is None else C.c_void_p(int(lower_src))
        hi = None if upper_src is None else C.c_void_p(int(upper_src))
        check(lib.spmvb_slab_spmv(self.h, _ptr(x_ghosted), _ptr(y), lo, hi, mode, _stream(stream)))

    def interior(self, x_ghosted, y, stream=None):
        check(lib.spmvb_slab_interior(self.h, _ptr(x_ghosted), _ptr(y), _stream(stream)))

    def boundary(self, x_ghosted, y, stream=None):
        check(lib.spmvb_slab_boundary(self.h, _ptr(x_ghosted), _ptr(y), _stream(stream)))

    @property
    def last_was_graph(self) -> bool:
        f = C.c_int32()
        check(lib.spmvb_slab_last_was_graph(self.h, C.byref(f)))
        return bool(f.value)


def ipc_export(dev_base) -> bytes:
    """CUDA IPC handle (64 bytes) of a vector from DeviceVector / spmvb_vec_alloc, for a neighbour process to map."""
    buf = C.create_string_buffer(64)
    check(lib.spmvb_ipc_export(_ptr(dev_base), buf))
    return buf.raw


def ipc_open(handle: bytes) -> int:
    p = C.c_void_p()
    check(lib.spmvb_ipc_open(C.create_string_buffer(handle, 64), C.byref(p)))
    return p.value


def ipc_close(ptr: int):
    check(lib.spmvb_ipc_close(C.c_void_p(ptr)))


class _Borrowed:
    """A device pointer owned by someone else."""

    def __init__(self, ptr, n):
        self.ptr, self.n = ptr, n

    def data_ptr(self):
        return self.ptr


class MultiSlab:
    """spmvb_multi_*: one host thread driving the z-slabs of a grid over a device list (devices may repeat)."""

    def __init__(self, spec: GridSpec, devices, fmt=FMT_PATTERN, diagonal=26.0, off_diagonal=-1.0, perturb=None,
                 values_in_pattern=True, min_pattern_rows=1, dict_cap=0, value_table_limit=256):
        validate_grid(spec)
        g = cabi.Grid(spec.nx, spec.ny, spec.nz, diagonal, off_diagonal, 0, 0, 0.0, 0.0)
        if perturb is not None:
            g.perturb, g.perturb_seed, g.perturb_fraction, g.perturb_noise = 1, perturb[0], perturb[1], perturb[2]
        o = _opts(value_table_limit, values_in_pattern, min_pattern_rows, dict_cap)
        devs = (C.c_int32 * len(devices))(*devices)
        h = C.c_void_p()
        check(lib.spmvb_multi_create(C.byref(g), fmt, C.byref(o), devs, len(devices), C.byref(h)))
        self.h, self.spec, self.n = h, spec, spec.rows()

    def __del__(self):
        if getattr(self, "h", None):
            lib.spmvb_multi_destroy(self.h)
            self.h = None

    @property
    def n_parts(self) -> int:
        c = C.c_int32()
        check(lib.spmvb_multi_parts(self.h, C.byref(c)))
        return c.value

    def part(self, g):
        """(device, z0, z1, matrix view, x_ghosted, y) of slab g; the views are owned by this object."""
        dev, z0, z1 = C.c_int32(), C.c_int64(), C.c_int64()
        a, x, y = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib.spmvb_multi_part(self.h, g, C.byref(dev), C.byref(z0), C.byref(z1), C.byref(a), C.byref(x), C.byref(y)))
        plane = self.spec.nx * self.spec.ny
        n = (z1.value - z0.value) * plane
        view = DeviceMatrix(a)
        view.__class__ = _BorrowedMatrix  # never destroyed from here
        return dev.value, z0.value, z1.value, view, _Borrowed(x.value, n + 2 * plane), _Borrowed(y.value, n)

    def fill_x(self, kind, seed=None, lo=0.0, hi=1.0):
        if kind == RANDOM and seed is None:
            raise InvalidArgument("seed is required for the random kind")
        check(lib.spmvb_multi_fill_x(self.h, kind, seed or 0, lo, hi))

    def upload_x(self, x):
        x = _np(x, np.float64)
        check(lib.spmvb_multi_upload_x(self.h, _ptr(x), x.shape[0]))

    def spmv(self, mode=SLAB_SERIAL):
        check(lib.spmvb_multi_spmv(self.h, mode))

    def sync(self):
        check(lib.spmvb_multi_sync(self.h))

    def download_y(self) -> np.ndarray:
        y = np.empty(self.n, dtype=np.float64)
        check(lib.spmvb_multi_download_y(self.h, _ptr(y), self.n))
        return y

    def bench(self, reps, mode=SLAB_SERIAL):
        """(host seconds between device-wide syncs, slowest slab's device seconds) for `reps` SpMVs incl. exchange."""
        t, td = C.c_double(), C.c_double()
        check(lib.spmvb_multi_bench(self.h, reps, mode, C.byref(t), C.byref(td)))
        return t.value, td.value


class _BorrowedMatrix(DeviceMatrix):
    def __del__(self):
        self.h = None
