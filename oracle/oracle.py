"""ctypes loader for the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_1612_00530_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

OK, INVALID_ARGUMENT, TABLE_OVERFLOW, INTEGRITY = 0, 1, 2, 3


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(OracleError):
    pass


class TableOverflowError(OracleError):  # errors.hpp:9
    pass


class IntegrityError(OracleError):  # errors.hpp:16
    pass


def build(force=False):
    src = os.path.join(_HERE, "spmvcomp_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-B", "liboracle.so"], check=True, capture_output=True)
    return _SO


class _Csr(C.Structure):
    _fields_ = [("n", C.c_int32), ("row_start", C.POINTER(C.c_int64)), ("cols", C.POINTER(C.c_int32)),
                ("vals", C.POINTER(C.c_double)), ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32)]


class _Perturb(C.Structure):
    _fields_ = [("enabled", C.c_int), ("seed", C.c_uint64), ("fraction", C.c_double), ("noise", C.c_double)]


class _Ell(C.Structure):
    _fields_ = [("n", C.c_int32), ("width", C.c_int32), ("nnz", C.c_int64), ("row_offset", C.c_int64),
                ("values", C.POINTER(C.c_double)), ("columns", C.POINTER(C.c_int32))]


class _Vt(C.Structure):
    _fields_ = [("n", C.c_int32), ("width", C.c_int32), ("m", C.c_int32), ("row_offset", C.c_int64),
                ("table", C.POINTER(C.c_double)), ("sorted_columns", C.POINTER(C.c_int32)),
                ("ends", C.POINTER(C.c_int32))]


class _Pattern(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("row_offset", C.c_int64),
                ("table", C.POINTER(C.c_double)), ("n_patterns", C.c_int32),
                ("disp_offsets", C.POINTER(C.c_int64)), ("disp_flat", C.POINTER(C.c_int32)),
                ("ends_flat", C.POINTER(C.c_int32)), ("row_pattern", C.POINTER(C.c_int32)),
                ("values_in_pattern", C.c_int), ("n_exc", C.c_int32), ("w_exc", C.c_int32),
                ("exc_rows", C.POINTER(C.c_int32)), ("exc_values", C.POINTER(C.c_double)),
                ("exc_columns", C.POINTER(C.c_int32))]


class Cost(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("bytes_per_row", "flops_per_row", "bytes_per_flop", "values",
                                          "indices", "ends", "pattern_id", "input_vector")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_SO)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_required_bandwidth.restype = C.c_double
        _lib.orc_roofline.restype = C.c_double
        _lib.orc_required_bandwidth.argtypes = [C.c_double, C.POINTER(Cost)]
        _lib.orc_roofline.argtypes = [C.POINTER(Cost), C.c_double, C.c_double, C.POINTER(C.c_int)]
        _lib.orc_generate_rows.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                           C.POINTER(_Perturb), C.c_int64, C.c_int64,
                                           C.POINTER(C.POINTER(_Csr))]
        _lib.orc_make_test_vector.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.c_double, C.c_double,
                                              C.c_int64, C.c_void_p]
        _lib.orc_compress_patterns_grid.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                                    C.POINTER(_Perturb), C.c_int, C.c_size_t, C.c_int32,
                                                    C.c_int32, C.POINTER(C.POINTER(_Pattern))]
        _lib.orc_to_ell.argtypes = [C.POINTER(_Csr), C.c_int32, C.c_int64, C.POINTER(C.POINTER(_Ell))]
        _lib.orc_compress_values.argtypes = [C.POINTER(_Csr), C.c_size_t, C.c_int32, C.c_int64,
                                             C.POINTER(C.POINTER(_Vt))]
        _lib.orc_compress_patterns.argtypes = [C.POINTER(_Csr), C.c_int, C.c_size_t, C.c_int32, C.c_int32,
                                               C.c_int64, C.POINTER(C.POINTER(_Pattern))]
        _lib.orc_scan_value_table.argtypes = [C.POINTER(_Csr), C.c_size_t, C.c_void_p, C.POINTER(C.c_int32)]
        _lib.orc_validate_vt.argtypes = [C.POINTER(_Vt), C.c_int64]
        _lib.orc_validate_pattern.argtypes = [C.POINTER(_Pattern), C.c_int64]
        for name, st in (("ell", _Ell), ("vt", _Vt), ("pattern", _Pattern)):
            getattr(_lib, f"orc_spmv_{name}").argtypes = [C.POINTER(st), C.c_void_p, C.c_int64, C.c_void_p,
                                                          C.c_int32, C.c_int32, C.c_int]
            getattr(_lib, f"orc_spmv_{name}").restype = None
        _lib.orc_spmv_csr.argtypes = [C.POINTER(_Csr), C.c_void_p, C.c_void_p]
        _lib.orc_spmv_csr.restype = None
        _lib.orc_row_abs_scale.argtypes = [C.POINTER(_Csr), C.c_void_p, C.c_void_p]
        _lib.orc_row_abs_scale.restype = None
        _lib.orc_dot.restype = C.c_double
        _lib.orc_dot.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        _lib.orc_waxpby.restype = None
        _lib.orc_waxpby.argtypes = [C.c_double, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_int64]
        _lib.orc_cg_solve.argtypes = [C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_double,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_void_p, C.POINTER(C.c_int32)]
        _lib.orc_csr_from_arrays.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.POINTER(C.POINTER(_Csr))]
    return _lib


def _check(rc):
    if rc == OK:
        return
    msg = lib().orc_last_error().decode()
    cls = {INVALID_ARGUMENT: InvalidArgument, TABLE_OVERFLOW: TableOverflowError,
           INTEGRITY: IntegrityError}.get(rc, OracleError)
    raise cls(rc, msg)


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(int(n),)).view(dtype)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class _Owned:
    _free = None

    def __init__(self, p):
        self.p = p

    def __del__(self):
        if getattr(self, "p", None) is not None and _lib is not None:
            getattr(_lib, self._free)(self.p)
            self.p = None

    @property
    def s(self):
        return self.p.contents


class Csr(_Owned):
    """StencilMatrix (stencil.hpp:19-36)."""
    _free = "orc_csr_free"

    n = property(lambda self: self.s.n)
    row_start = property(lambda self: _arr(self.s.row_start, self.s.n + 1, np.int64))
    nnz = property(lambda self: int(self.row_start[self.s.n]))
    cols = property(lambda self: _arr(self.s.cols, self.nnz, np.int32))
    vals = property(lambda self: _arr(self.s.vals, self.nnz, np.float64))

    def row(self, i):
        b, e = self.row_start[i], self.row_start[i + 1]
        return self.cols[b:e], self.vals[b:e]

    def __eq__(self, other):
        return bool(lib().orc_csr_equal(self.p, other.p))

    def dense(self, n_cols=None):
        n_cols = n_cols or self.n
        d = np.zeros((self.n, n_cols))
        rs = self.row_start
        for i in range(self.n):
            d[i, self.cols[rs[i]:rs[i + 1]]] = self.vals[rs[i]:rs[i + 1]]
        return d


class Ell(_Owned):
    _free = "orc_ell_free"
    n = property(lambda self: self.s.n)
    width = property(lambda self: self.s.width)
    nnz = property(lambda self: self.s.nnz)
    row_offset = property(lambda self: self.s.row_offset)
    values = property(lambda self: _arr(self.s.values, self.s.n * self.s.width, np.float64))
    columns = property(lambda self: _arr(self.s.columns, self.s.n * self.s.width, np.int32))


class Vt(_Owned):
    _free = "orc_vt_free"
    n = property(lambda self: self.s.n)
    width = property(lambda self: self.s.width)
    m = property(lambda self: self.s.m)
    row_offset = property(lambda self: self.s.row_offset)
    table = property(lambda self: _arr(self.s.table, self.s.m, np.float64))
    sorted_columns = property(lambda self: _arr(self.s.sorted_columns, self.s.n * self.s.width, np.int32))
    ends = property(lambda self: _arr(self.s.ends, self.s.n * self.s.m, np.int32))


class Pattern(_Owned):
    _free = "orc_pattern_free"
    n = property(lambda self: self.s.n)
    m = property(lambda self: self.s.m)
    row_offset = property(lambda self: self.s.row_offset)
    table = property(lambda self: _arr(self.s.table, self.s.m, np.float64))
    n_patterns = property(lambda self: self.s.n_patterns)
    disp_offsets = property(lambda self: _arr(self.s.disp_offsets, self.s.n_patterns + 1, np.int64))
    disp_flat = property(lambda self: _arr(self.s.disp_flat, self.disp_offsets[-1], np.int32))
    ends_flat = property(lambda self: _arr(self.s.ends_flat, self.s.n_patterns * self.s.m, np.int32))
    row_pattern = property(lambda self: _arr(self.s.row_pattern, self.s.n, np.int32))
    values_in_pattern = property(lambda self: bool(self.s.values_in_pattern))
    n_exc = property(lambda self: self.s.n_exc)
    w_exc = property(lambda self: self.s.w_exc)
    exc_rows = property(lambda self: _arr(self.s.exc_rows, self.s.n_exc, np.int32))
    exc_values = property(lambda self: _arr(self.s.exc_values, self.s.n_exc * self.s.w_exc, np.float64))
    exc_columns = property(lambda self: _arr(self.s.exc_columns, self.s.n_exc * self.s.w_exc, np.int32))

    def pattern(self, p):
        o = self.disp_offsets
        return self.disp_flat[o[p]:o[p + 1]].tolist(), self.ends_flat[p * self.m:(p + 1) * self.m].tolist()


def _pert(perturb):
    if perturb is None:
        return None
    seed, fraction, noise = perturb
    return C.byref(_Perturb(1, seed, fraction, noise))


def generate_matrix(nx, ny, nz, diagonal=26.0, off_diagonal=-1.0, perturb=None, row_begin=0, row_end=None):
    """stencil.hpp:40-45.  perturb=(seed, fraction, noise) enables the config-4 recipe."""
    out = C.POINTER(_Csr)()
    if row_end is None:
        row_end = nx * ny * nz
    _check(lib().orc_generate_rows(nx, ny, nz, diagonal, off_diagonal, _pert(perturb), row_begin, row_end,
                                   C.byref(out)))
    return Csr(out)


def stencil_from_rows(n, rows):
    """stencil.hpp:47-50; rows = list of lists of (col, value)."""
    rs = np.zeros(n + 1, dtype=np.int64)
    cols, vals = [], []
    for i, r in enumerate(rows):
        rs[i + 1] = rs[i] + len(r)
        cols += [c for c, _ in r]
        vals += [v for _, v in r]
    cols = np.asarray(cols, dtype=np.int32)
    vals = np.asarray(vals, dtype=np.float64)
    out = C.POINTER(_Csr)()
    _check(lib().orc_csr_from_arrays(n, _ptr(rs), _ptr(cols), _ptr(vals), C.byref(out)))
    return Csr(out)


def csr_from_arrays(n, row_start, cols, vals):
    row_start = np.ascontiguousarray(row_start, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    out = C.POINTER(_Csr)()
    _check(lib().orc_csr_from_arrays(n, _ptr(row_start), _ptr(cols), _ptr(vals), C.byref(out)))
    return Csr(out)


def is_symmetric(m):
    return bool(lib().orc_is_symmetric(m.p))


ONES, LINEAR, RANDOM = 0, 1, 2


def make_test_vector(n, kind, seed=None, lo=0.0, hi=1.0, first_index=0):
    """stencil.hpp:54-59; random needs a seed; [lo,hi) defaults to the header's [0,1)."""
    if kind == RANDOM and seed is None:
        raise InvalidArgument(INVALID_ARGUMENT, "seed is required for the random kind")
    out = np.empty(max(n, 0), dtype=np.float64)
    _check(lib().orc_make_test_vector(n, kind, seed or 0, lo, hi, first_index, _ptr(out)))
    return out


def to_ell(m, min_width=0, row_offset=0):
    out = C.POINTER(_Ell)()
    _check(lib().orc_to_ell(m.p, min_width, row_offset, C.byref(out)))
    return Ell(out)


def to_stencil(a):
    out = C.POINTER(_Csr)()
    _check(lib().orc_ell_to_csr(a.p, C.byref(out)))
    return Csr(out)


def scan_value_table(m, limit=256):
    tab = np.empty(limit + 1, dtype=np.float64)
    k = C.c_int32()
    _check(lib().orc_scan_value_table(m.p, limit, _ptr(tab), C.byref(k)))
    return tab[:k.value].copy()


def compress_values(m, limit=256, min_width=0, row_offset=0):
    out = C.POINTER(_Vt)()
    _check(lib().orc_compress_values(m.p, limit, min_width, row_offset, C.byref(out)))
    return Vt(out)


def compress_patterns(m, values_in_pattern=False, limit=256, min_pattern_rows=1, dict_cap=0, row_offset=0):
    out = C.POINTER(_Pattern)()
    _check(lib().orc_compress_patterns(m.p, int(values_in_pattern), limit, min_pattern_rows, dict_cap, row_offset,
                                       C.byref(out)))
    return Pattern(out)


def compress_patterns_grid(nx, ny, nz, diagonal=26.0, off_diagonal=-1.0, perturb=None,
                           values_in_pattern=False, limit=256, min_pattern_rows=1, dict_cap=0):
    out = C.POINTER(_Pattern)()
    _check(lib().orc_compress_patterns_grid(nx, ny, nz, diagonal, off_diagonal, _pert(perturb),
                                            int(values_in_pattern), limit, min_pattern_rows, dict_cap,
                                            C.byref(out)))
    return Pattern(out)


def validate(c, n_cols=None):
    n_cols = c.n if n_cols is None else n_cols
    if isinstance(c, Vt):
        _check(lib().orc_validate_vt(c.p, n_cols))
    else:
        _check(lib().orc_validate_pattern(c.p, n_cols))


def decompress(c):
    out = C.POINTER(_Csr)()
    if isinstance(c, Vt):
        _check(lib().orc_decompress_vt(c.p, C.byref(out)))
    else:
        _check(lib().orc_decompress_pattern(c.p, C.byref(out)))
    return Csr(out)


def spmv_rows(a, x, y, begin, end, x_col0=0, threads=1):
    """unchecked::spmv_rows (kernels.hpp:27-36)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    assert y.dtype == np.float64 and y.flags.c_contiguous
    fn = {Ell: "orc_spmv_ell", Vt: "orc_spmv_vt", Pattern: "orc_spmv_pattern"}[type(a)]
    getattr(lib(), fn)(a.p, _ptr(x), x_col0, _ptr(y), begin, end, threads)


def spmv(a, x, threads=1):
    """spmv (kernels.hpp:19-25): validated, returns a fresh vector."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if isinstance(a, Csr):
        if x.shape[0] != a.n:
            raise InvalidArgument(INVALID_ARGUMENT, "length mismatch")
        y = np.empty(a.n)
        lib().orc_spmv_csr(a.p, _ptr(x), _ptr(y))
        return y
    if x.shape[0] != a.n:
        raise InvalidArgument(INVALID_ARGUMENT, f"x has {x.shape[0]} entries, matrix has {a.n} rows")
    if not isinstance(a, Ell):
        validate(a)
    y = np.empty(a.n)
    spmv_rows(a, x, y, 0, a.n, 0, threads)
    return y


def row_abs_scale(m, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    s = np.empty(m.n)
    lib().orc_row_abs_scale(m.p, _ptr(x), _ptr(s))
    return s


FMT_ELL, FMT_VT, FMT_PATTERN, FMT_PATTERN_VALUES = 0, 1, 2, 3


def format_cost(fmt, row_nnz, table_size, include_input_vector=False):
    c = Cost()
    _check(lib().orc_format_cost(fmt, row_nnz, table_size, int(include_input_vector), C.byref(c)))
    return c


def required_bandwidth(flops_per_second, cost):
    return lib().orc_required_bandwidth(flops_per_second, C.byref(cost))


def roofline(cost, read_bandwidth=75e9, peak_flops=None):
    lim = C.c_int()
    f = lib().orc_roofline(C.byref(cost), read_bandwidth, peak_flops or 0.0, C.byref(lim))
    return f, ("compute" if lim.value else "bandwidth")


def measured_cost(a):
    c = Cost()
    fn = {Ell: "orc_measured_cost_ell", Vt: "orc_measured_cost_vt", Pattern: "orc_measured_cost_pattern"}[type(a)]
    _check(getattr(lib(), fn)(a.p, C.byref(c)))
    return c


def dot(u, v):
    """dot (kernels.hpp:39): index-ascending sum."""
    u, v = np.ascontiguousarray(u, dtype=np.float64), np.ascontiguousarray(v, dtype=np.float64)
    if u.shape != v.shape:
        raise InvalidArgument(INVALID_ARGUMENT, "length mismatch")
    return lib().orc_dot(_ptr(u), _ptr(v), u.shape[0])


def waxpby(alpha, x, beta, y):
    """waxpby (kernels.hpp:41)."""
    x, y = np.ascontiguousarray(x, dtype=np.float64), np.ascontiguousarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise InvalidArgument(INVALID_ARGUMENT, "length mismatch")
    w = np.empty_like(x)
    lib().orc_waxpby(alpha, _ptr(x), beta, _ptr(y), _ptr(w), x.shape[0])
    return w


class DivergenceError(OracleError):  # errors.hpp:22
    pass


def symgs_sweep(m, x, b):
    """symgs_sweep (kernels.hpp:44-48): forward then backward Gauss-Seidel sweep in natural order; returns the new x."""
    x = np.array(x, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if x.shape[0] != m.n or b.shape[0] != m.n:
        raise InvalidArgument(INVALID_ARGUMENT, "length mismatch")
    fn = lib().orc_symgs_sweep
    fn.argtypes, fn.restype = [C.c_void_p, C.c_void_p, C.c_void_p], C.c_int
    _check(fn(C.cast(m.p, C.c_void_p), _ptr(x), _ptr(b)))
    return x


def cg_solve(a, b, max_iterations=500, tolerance=1e-8, symgs_sweeps=0, matrix=None):
    """cg_solve (solver.hpp:40-46); `a` is the SpMV backend (Ell, Vt or Pattern).  symgs_sweeps >= 1 preconditions with
    that many SymGS sweeps from a zero guess on `matrix` (the Csr).  Returns (x, iterations, converged, residual_history)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.shape[0] != a.n:
        raise InvalidArgument(INVALID_ARGUMENT, "length mismatch")
    fmt = {Ell: 0, Vt: 1, Pattern: 2}[type(a)]
    x = np.empty(a.n)
    hist = np.zeros(max_iterations + 1)
    it, conv, div = C.c_int32(), C.c_int32(), C.c_int32()
    if symgs_sweeps:
        fn = lib().orc_pcg_solve
        fn.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_int32,
                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        fn.restype = C.c_int
        _check(fn(fmt, C.cast(a.p, C.c_void_p), C.cast(matrix.p, C.c_void_p), a.n, _ptr(b), _ptr(x), max_iterations, tolerance,
                  symgs_sweeps, C.byref(it), C.byref(conv), _ptr(hist), C.byref(div)))
    else:
        _check(lib().orc_cg_solve(fmt, C.cast(a.p, C.c_void_p), a.n, _ptr(b), _ptr(x), max_iterations, tolerance,
                                  C.byref(it), C.byref(conv), _ptr(hist), C.byref(div)))
    if div.value:
        raise DivergenceError(6, f"non-finite value in iteration {div.value}")
    return x, it.value, bool(conv.value), hist[:it.value + 1].copy()
