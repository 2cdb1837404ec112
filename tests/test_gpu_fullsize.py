"""Parity at BASELINE.json's full sizes, inside the suite:
  * 256^3 (configs[2], one GPU): the device-built id stream and y against the CPU oracle, bit for bit, every row;
  * 512^3 (configs[4] at one GPU): the host cannot hold that matrix, so the oracle regenerates and compresses chunks of 8
    planes (2.1 M rows each) of the global grid and the ids (through the dictionaries) and y of those chunks are compared
    (SURVEY H4);
  * the reference-signature call spmv(fmt, Vector) -- upload the struct's arrays, validate, x in / y out through pageable
    host memory -- as the C++ shim issues it (paper_1612_00530_b200/cpp/spmvcomp_host.cpp:spmv_checked), at 128^3.
Size-independent properties ride along: linearity and A*ones >= 0 with exact zeros on interior rows."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 7


@pytest.fixture(scope="module")
def sp():
    import paper_1612_00530_b200 as sp
    assert sp.device_count() >= 1
    return sp


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def test_256_cubed_ids_and_y_equal_the_oracle(sp, orc):
    g = (256, 256, 256)
    cores = os.cpu_count() or 1
    ref = orc.compress_patterns_grid(*g, values_in_pattern=True)
    n = ref.n
    x = orc.make_test_vector(n, orc.RANDOM, seed=SEED, lo=-1.0, hi=1.0)
    y_ref = np.zeros(n)
    orc.spmv_rows(ref, x, y_ref, 0, n, threads=cores)
    dev = sp.compress_patterns(sp.generate_matrix(sp.GridSpec(*g)), True)
    assert dev.info.n_patterns == 27
    assert np.array_equal(dev.download("row_pattern"), ref.row_pattern)
    assert dev.download("disp_flat").tobytes() == ref.disp_flat.tobytes()
    assert dev.download("ends_flat").tobytes() == ref.ends_flat.tobytes()
    dx, dy = sp.DeviceVector(n), sp.DeviceVector.from_host(np.full(n, np.nan))
    sp.check(sp.lib.spmvb_vec_fill(dx.ptr, n, sp.RANDOM, SEED, -1.0, 1.0, 0, None))  # the device's own fill of the seeded vector
    assert np.array_equal(bits(dx.to_host()), bits(x))
    sp.spmv_rows(dev, dx, dy, 0, n)
    assert sp.get_option("last_pattern_kernel") == 9  # the tensor-ring kernel: the one bench.py times
    y = dy.to_host()
    assert int((bits(y) != bits(y_ref)).sum()) == 0
    # A * ones: exact zeros on the interior rows, >= 0 everywhere
    ones = sp.DeviceVector.from_host(np.ones(n))
    sp.spmv_rows(dev, ones, dy, 0, n)
    y1 = dy.to_host().reshape(g[2], g[1], g[0])
    assert np.all(y1[1:-1, 1:-1, 1:-1] == 0.0) and y1.min() >= 0.0 and y1[0, 0, 0] == 19.0
    # linearity: A(2x + ones) against 2 Ax + A ones, scaled by sum |a_ik x_k| <= 52 * 3
    sp.spmv_rows(dev, sp.DeviceVector.from_host(2.0 * x + 1.0), dy, 0, n)
    assert np.abs(dy.to_host() - (2.0 * y + y1.ravel())).max() <= 1e-12 * 52 * 3


def test_512_cubed_chunks_equal_the_oracle(sp, orc):
    g = (512, 512, 512)
    cores = os.cpu_count() or 1
    n = g[0] * g[1] * g[2]
    plane = g[0] * g[1]
    big = sp.MultiSlab(sp.GridSpec(*g), [0])  # device-side build in one piece: generator -> compressor, the CSR is freed
    _, _, _, a, xg, yg = big.part(0)
    big.fill_x(sp.RANDOM, SEED, -1.0, 1.0)
    big.spmv(sp.SLAB_SERIAL)  # one slab: a single launch over all planes, on the slab's own stream
    big.sync()
    assert sp.get_option("last_pattern_kernel") == 9
    yd = big.download_y()
    ids = a.download("row_pattern")
    off, flat = a.download("disp_offsets"), a.download("disp_flat")
    shapes = [tuple(flat[off[q]:off[q + 1]].tolist()) for q in range(a.info.n_patterns)]
    assert len(shapes) == 27
    for z0 in (0, 131, 300, g[2] - 8):  # the first and last planes and two chunks inside
        r0, r1 = z0 * plane, (z0 + 8) * plane
        co = orc.compress_patterns(orc.generate_matrix(*g, row_begin=r0, row_end=r1), True, row_offset=r0)
        oshapes = [tuple(co.disp_flat[co.disp_offsets[q]:co.disp_offsets[q + 1]].tolist()) for q in range(len(co.disp_offsets) - 1)]
        to_dev = np.array([shapes.index(s) for s in oshapes], dtype=np.int32)  # chunk numbering -> whole-matrix numbering
        assert np.array_equal(to_dev[co.row_pattern], ids[r0:r1]), f"ids differ in planes [{z0},{z0 + 8})"
        lo, hi = max(r0 - plane, 0), min(r1 + plane, n)
        xl = orc.make_test_vector(hi - lo, orc.RANDOM, seed=SEED, lo=-1.0, hi=1.0, first_index=lo)
        yo = np.zeros(r1 - r0)
        orc.spmv_rows(co, xl, yo, 0, r1 - r0, x_col0=lo, threads=cores)
        assert int((bits(yo) != bits(yd[r0:r1])).sum()) == 0, f"y differs in planes [{z0},{z0 + 8})"
    # a checksum with a closed form: for x = ones, y_i = 26 - (nnz_i - 1), small integers, so sum(y) = 27 n - nnz exactly,
    # and the interior rows (27 entries) are exactly zero
    big.fill_x(sp.ONES)
    big.spmv(sp.SLAB_SERIAL)
    big.sync()
    y1 = big.download_y()
    nnz = (3 * g[0] - 2) * (3 * g[1] - 2) * (3 * g[2] - 2)
    assert a.info.nnz == nnz and float(y1.sum()) == float(27 * n - nnz)
    y1 = y1.reshape(g[2], g[1], g[0])
    assert np.all(y1[1:-1, 1:-1, 1:-1] == 0.0) and y1.min() >= 0.0
    del big


def test_reference_signature_call_with_pageable_vectors(sp, orc):
    """spmv(const PatternCompressedMatrix&, const Vector&) -> Vector as the shim runs it: the struct's arrays uploaded byte for
    byte, validated, x and y through pageable host buffers (spmvb_spmv_host pipelines the copies)."""
    g = (128, 128, 128)
    ref = orc.compress_patterns_grid(*g, values_in_pattern=True)
    x = orc.make_test_vector(ref.n, orc.RANDOM, seed=SEED, lo=-1.0, hi=1.0)  # pageable numpy memory
    y_ref = orc.spmv(ref, x, threads=os.cpu_count() or 1)
    for _ in range(2):
        d = sp.upload_pattern(ref.n, ref.table, ref.disp_offsets, ref.disp_flat, ref.ends_flat, ref.row_pattern, True)
        sp.check(sp.lib.spmvb_validate(d.h, ref.n, None))
        y = np.empty(ref.n)
        sp.check(sp.lib.spmvb_spmv_host(d.h, x.ctypes.data, ref.n, y.ctypes.data))
        assert int((bits(y) != bits(y_ref)).sum()) == 0
        del d
    with pytest.raises(sp.InvalidArgument):  # length mismatch
        d = sp.upload_pattern(ref.n, ref.table, ref.disp_offsets, ref.disp_flat, ref.ends_flat, ref.row_pattern, True)
        sp.check(sp.lib.spmvb_spmv_host(d.h, x.ctypes.data, ref.n - 1, np.empty(ref.n).ctypes.data))


@pytest.mark.parametrize("g", [(128, 128, 64), (64, 64, 64), (128, 128, 65)])
def test_pageable_host_vectors_are_staged(sp, orc, g):
    """spmvb_spmv_host with pageable x / y ("host_stage"): pinned bounce buffers filled and drained by host threads inside the
    chunk pipeline (>= 1 M rows) or around the plain copy-run-copy path -- the same bits as the driver's pageable copies and
    as pinned buffers, for every format; repeated calls reuse the buffers."""
    import torch
    ref = orc.compress_patterns_grid(*g, values_in_pattern=True)
    n = ref.n
    x = orc.make_test_vector(n, orc.RANDOM, seed=SEED, lo=-1.0, hi=1.0)
    y_ref = orc.spmv(ref, x, threads=os.cpu_count() or 1)
    d = sp.upload_pattern(ref.n, ref.table, ref.disp_offsets, ref.disp_flat, ref.ends_flat, ref.row_pattern, True)
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.empty(n, dtype=torch.float64).pin_memory()
    try:
        for stage, threads in ((1, 0), (1, 1), (1, 7), (0, 0), (1, 0)):
            sp.set_option("host_stage", stage)
            sp.set_option("host_copy_threads", threads)
            y = np.full(n, np.nan)
            sp.check(sp.lib.spmvb_spmv_host(d.h, x.ctypes.data, n, y.ctypes.data))            # pageable in, pageable out
            assert int((bits(y) != bits(y_ref)).sum()) == 0, (stage, threads)
            y2 = np.full(n, np.nan)
            sp.check(sp.lib.spmvb_spmv_host(d.h, xp.data_ptr(), n, y2.ctypes.data))            # pinned in, pageable out
            assert int((bits(y2) != bits(y_ref)).sum()) == 0
            yp.fill_(float("nan"))
            sp.check(sp.lib.spmvb_spmv_host(d.h, x.ctypes.data, n, yp.data_ptr()))             # pageable in, pinned out
            assert int((bits(yp.numpy()) != bits(y_ref)).sum()) == 0
    finally:
        sp.set_option("host_stage", 1)
        sp.set_option("host_copy_threads", 0)
    ell = orc.to_ell(orc.generate_matrix(*g)) if n <= 300000 else None
    if ell is not None:  # a format without a known reach: the plain path
        de = sp.upload_ell(ell.n, ell.width, ell.nnz, ell.values, ell.columns)
        y = np.full(n, np.nan)
        sp.check(sp.lib.spmvb_spmv_host(de.h, x.ctypes.data, n, y.ctypes.data))
        assert int((bits(y) != bits(orc.spmv(ell, x))).sum()) == 0
