"""TEST INFRASTRUCTURE (oracle): numpy restatement of the file formats either side of the SpMV path.

Binary serialization as SPEC.md:186 words it -- little-endian, a 16-byte magic + version header, the fields in
declaration order (stencil.hpp:18-23, ell.hpp:14-19, compress.hpp:36-41,65-70), 8-byte length prefixes for variable
arrays -- with the concrete bytes this repository chose (include/spmvcomp/io.hpp; the reference does not ship its layout
document: "parity unpinned").  Matrix Market export as stencil.hpp:61-64 describes it.  Only tests/ import this module.
"""
import struct

import numpy as np

MAGIC = b"SPMVCOMP"
VERSION = 1
KIND_STENCIL, KIND_ELL, KIND_VT, KIND_PATTERN = 1, 2, 3, 4


def _hdr(kind):
    return MAGIC + struct.pack("<II", VERSION, kind)


def _vec(a, dtype):
    a = np.ascontiguousarray(a, dtype=np.dtype(dtype).newbyteorder("<"))
    return struct.pack("<Q", a.size) + a.tobytes()


def dump_stencil(m, grid=(0, 0, 0)):
    """StencilMatrix: n, row_start, cols, vals, grid (nx, ny, nz)."""
    return (_hdr(KIND_STENCIL) + struct.pack("<i", m.n) + _vec(m.row_start, "i8") + _vec(m.cols, "i4") + _vec(m.vals, "f8")
            + struct.pack("<iii", *grid))


def dump_ell(a):
    """EllMatrix: n, width, nnz, values, columns."""
    return _hdr(KIND_ELL) + struct.pack("<iiq", a.n, a.width, a.nnz) + _vec(a.values, "f8") + _vec(a.columns, "i4")


def dump_vt(a):
    """VtCompressedMatrix: n, width, table, sorted_columns, ends."""
    return _hdr(KIND_VT) + struct.pack("<ii", a.n, a.width) + _vec(a.table, "f8") + _vec(a.sorted_columns, "i4") + _vec(a.ends, "i4")


def dump_pattern(a):
    """PatternCompressedMatrix: n, table, patterns (each: displacements, ends), row_pattern, values_in_pattern and,
    when the ends are not folded into the table, the ends of every row (compress.hpp:62-64)."""
    out = [_hdr(KIND_PATTERN), struct.pack("<i", a.n), _vec(a.table, "f8"), struct.pack("<Q", a.n_patterns)]
    pats = [a.pattern(p) for p in range(a.n_patterns)]
    for disp, ends in pats:
        out += [_vec(disp, "i4"), _vec(ends, "i4")]
    out += [_vec(a.row_pattern, "i4"), struct.pack("<B", 1 if a.values_in_pattern else 0)]
    if not a.values_in_pattern:
        ends = np.array([e for _, e in pats], dtype=np.int32).reshape(a.n_patterns, a.m)
        out.append(_vec(ends[np.asarray(a.row_pattern)].reshape(-1), "i4"))
    return b"".join(out)


class _Cursor:
    def __init__(self, data):
        self.d, self.o = data, 0

    def take(self, fmt):
        v = struct.unpack_from("<" + fmt, self.d, self.o)
        self.o += struct.calcsize("<" + fmt)
        return v if len(v) > 1 else v[0]

    def vec(self, dtype):
        n = self.take("Q")
        dt = np.dtype(dtype).newbyteorder("<")
        a = np.frombuffer(self.d, dtype=dt, count=n, offset=self.o)
        self.o += n * dt.itemsize
        return a


def parse(data):
    """Bytes of any of the four files -> dict of its fields (raises ValueError on a malformed header or length)."""
    if data[:8] != MAGIC:
        raise ValueError("bad magic")
    c = _Cursor(data)
    c.o = 8
    version, kind = c.take("II")
    if version != VERSION:
        raise ValueError("bad version")
    if kind == KIND_STENCIL:
        out = dict(kind=kind, n=c.take("i"), row_start=c.vec("i8"), cols=c.vec("i4"), vals=c.vec("f8"), grid=c.take("iii"))
    elif kind == KIND_ELL:
        n, width, nnz = c.take("iiq")
        out = dict(kind=kind, n=n, width=width, nnz=nnz, values=c.vec("f8"), columns=c.vec("i4"))
    elif kind == KIND_VT:
        n, width = c.take("ii")
        out = dict(kind=kind, n=n, width=width, table=c.vec("f8"), sorted_columns=c.vec("i4"), ends=c.vec("i4"))
    elif kind == KIND_PATTERN:
        out = dict(kind=kind, n=c.take("i"), table=c.vec("f8"))
        out["patterns"] = [(c.vec("i4"), c.vec("i4")) for _ in range(c.take("Q"))]
        out["row_pattern"] = c.vec("i4")
        out["values_in_pattern"] = bool(c.take("B"))
        if not out["values_in_pattern"]:
            out["row_ends"] = c.vec("i4")
    else:
        raise ValueError("bad kind")
    if c.o != len(data):
        raise ValueError("trailing bytes")
    return out


def payload_bytes_per_row(data):
    """What measured_cost counts (perf_model.hpp:74-77): the streamed arrays only -- no header, scalars, length
    prefixes or value table; pattern tables amortised over the rows."""
    f = parse(data)
    n = f["n"]
    if f["kind"] == KIND_ELL:
        return (f["values"].nbytes + f["columns"].nbytes) / n
    if f["kind"] == KIND_VT:
        return (f["sorted_columns"].nbytes + f["ends"].nbytes) / n
    if f["kind"] == KIND_PATTERN:
        table = sum(d.nbytes for d, _ in f["patterns"])
        ends = f["row_ends"].nbytes if not f["values_in_pattern"] else sum(e.nbytes for _, e in f["patterns"])
        return (f["row_pattern"].nbytes + table + ends) / n
    raise ValueError("no byte model for this kind")


def matrix_market_text(m):
    """stencil.hpp:61-64: coordinate real symmetric, 1-based, lower triangle only, 17 significant digits."""
    rs, cols, vals = m.row_start, m.cols, m.vals
    lines = []
    for i in range(m.n):
        for t in range(rs[i], rs[i + 1]):
            if cols[t] <= i:
                lines.append("%d %d %.17g\n" % (i + 1, cols[t] + 1, vals[t]))
    return "%%MatrixMarket matrix coordinate real symmetric\n" + "%d %d %d\n" % (m.n, m.n, len(lines)) + "".join(lines)
