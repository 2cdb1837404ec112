"""GPU parity tests for the device-side generator / compressor: every stream the
CUDA builders produce is compared byte for byte with the CPU oracle's."""
import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRIDS = [(1, 1, 1), (2, 2, 2), (3, 3, 3), (4, 4, 4), (5, 4, 3), (2, 5, 1), (7, 1, 4), (8, 3, 2), (6, 6, 6),
         (33, 9, 5), (40, 37, 11), (32, 32, 32)]
PERT = (11, 0.1, 0.1)


@pytest.fixture(scope="module")
def sp():
    import paper_1612_00530_b200 as sp
    return sp


def same(a, b):
    return np.ascontiguousarray(a).tobytes() == np.ascontiguousarray(b).tobytes()


def assert_csr(dev, ref):
    assert dev.n == ref.n and dev.nnz == ref.nnz
    assert same(dev.download("row_start"), ref.row_start)
    assert same(dev.download("cols"), ref.cols)
    assert same(dev.download("vals"), ref.vals)


def assert_pattern(dev, ref):
    i = dev.info
    assert (i.n, i.m, i.n_patterns, i.n_exc, i.w_exc) == (ref.n, ref.m, ref.n_patterns, ref.n_exc, ref.w_exc)
    for f in ("table", "row_pattern", "disp_offsets", "disp_flat", "ends_flat", "exc_rows", "exc_values", "exc_columns"):
        assert same(dev.download(f), getattr(ref, f)), f


@pytest.mark.parametrize("g", GRIDS)
def test_generate_and_formats(sp, orc, g):
    spec = sp.GridSpec(*g)
    ref = orc.generate_matrix(*g)
    m = sp.generate_matrix(spec)
    assert_csr(m, ref)
    ell, e_ref = sp.to_ell(m), orc.to_ell(ref)
    assert (ell.info.width, ell.info.nnz) == (e_ref.width, e_ref.nnz)
    assert same(ell.download("values"), e_ref.values) and same(ell.download("columns"), e_ref.columns)
    vt, v_ref = sp.compress_values(m), orc.compress_values(ref)
    assert (vt.info.width, vt.info.m) == (v_ref.width, v_ref.m)
    for f in ("table", "sorted_columns", "ends"):
        assert same(vt.download(f), getattr(v_ref, f)), f
    for vip in (False, True):
        assert_pattern(sp.compress_patterns(m, vip), orc.compress_patterns(ref, vip))
    # decompress / to_stencil on the device: exact round trip
    for c in (ell, vt, sp.compress_patterns(m)):
        sp.validate(c)
        assert_csr(sp.decompress(c), ref)


def test_round_trip_all_small_grids(sp, orc):
    """Acceptance criterion 4 on the device for nx,ny,nz in [1,4]."""
    for g in itertools.product(range(1, 5), repeat=3):
        m = sp.generate_matrix(sp.GridSpec(*g))
        ref = orc.generate_matrix(*g)
        pc = sp.compress_patterns(m)
        assert pc.info.n_patterns == min(g[0], 3) * min(g[1], 3) * min(g[2], 3)
        assert_csr(sp.decompress(pc), ref)
        assert_csr(sp.decompress(sp.compress_values(m)), ref)


@pytest.mark.parametrize("g", [(4, 4, 4), (16, 16, 16), (48, 40, 36)])
def test_perturbed_generator_and_hybrid(sp, orc, g):
    ref = orc.generate_matrix(*g, perturb=PERT)
    m = sp.generate_matrix(sp.GridSpec(*g), perturb=PERT)
    assert_csr(m, ref)
    e_ref = orc.to_ell(ref)
    ell = sp.to_ell(m)
    assert ell.info.width == e_ref.width and same(ell.download("values"), e_ref.values)
    assert same(ell.download("columns"), e_ref.columns)
    p_ref = orc.compress_patterns(ref, True, min_pattern_rows=2)
    pc = sp.compress_patterns(m, True, min_pattern_rows=2)
    assert_pattern(pc, p_ref)
    sp.validate(pc)
    assert_csr(sp.decompress(pc), ref)
    if g[0] >= 16:
        # the reference scheme cannot hold this matrix: noise makes every value distinct
        with pytest.raises(sp.TableOverflowError):
            sp.compress_values(m)
        with pytest.raises(sp.TableOverflowError):
            sp.compress_patterns(m)
    # dictionary cap: only the most frequent shapes stay, the rest become exception rows
    capped_ref = orc.compress_patterns(ref, True, min_pattern_rows=2, dict_cap=5)
    assert_pattern(sp.compress_patterns(m, True, min_pattern_rows=2, dict_cap=5), capped_ref)
    x = orc.make_test_vector(ref.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    for dev, r in ((pc, p_ref), (sp.compress_patterns(m, True, min_pattern_rows=2, dict_cap=5), capped_ref)):
        assert same(sp.spmv(dev, x), orc.spmv(r, x))


def test_slab_generation(sp, orc):
    """Global rows [r0,r1): columns stay global, ELL padding = own global row."""
    g = (12, 10, 9)
    plane = g[0] * g[1]
    for z0, z1 in ((0, 3), (3, 7), (7, 9)):
        ref = orc.generate_matrix(*g, row_begin=z0 * plane, row_end=z1 * plane)
        m = sp.generate_matrix(sp.GridSpec(*g), row_begin=z0 * plane, row_end=z1 * plane)
        assert_csr(m, ref)
        assert m.info.row_offset == z0 * plane
        e_ref = orc.to_ell(ref, min_width=27, row_offset=z0 * plane)
        ell = sp.to_ell(m, min_width=27)
        assert same(ell.download("values"), e_ref.values) and same(ell.download("columns"), e_ref.columns)
        v_ref = orc.compress_values(ref, min_width=27, row_offset=z0 * plane)
        vt = sp.compress_values(m, min_width=27)
        assert same(vt.download("sorted_columns"), v_ref.sorted_columns) and same(vt.download("ends"), v_ref.ends)


def test_explicit_rows_and_errors(sp, orc):
    rows = [[(i, 26.0)] for i in range(66)]
    rows[50] = [(45, -1.0), (49, -1.0), (50, 26.0), (51, -1.0), (65, -1.0)]
    m = sp.stencil_from_rows(66, rows)
    vt = sp.compress_values(m)
    assert vt.download("table").tolist() == [-1.0, 26.0]
    assert vt.download("sorted_columns")[50 * 5:51 * 5].tolist() == [45, 49, 51, 65, 50]
    assert vt.download("ends")[100:102].tolist() == [4, 5]
    pc = sp.compress_patterns(m)
    pid = pc.download("row_pattern")[50]
    off = pc.download("disp_offsets")
    assert pc.download("disp_flat")[off[pid]:off[pid + 1]].tolist() == [-5, -1, 1, 15, 0]
    assert pc.download("ends_flat")[pid * 2:pid * 2 + 2].tolist() == [4, 5]
    assert sp.spmv(pc, np.ones(66))[50] == 22.0
    with pytest.raises(sp.InvalidArgument):  # columns must be strictly ascending (stencil.hpp:47-48)
        sp.stencil_from_rows(2, [[(1, 1.0), (0, 1.0)], [(1, 1.0)]])
    with pytest.raises(sp.InvalidArgument):
        sp.stencil_from_rows(2, [[(0, 1.0), (2, 1.0)], [(1, 1.0)]])
    with pytest.raises(sp.InvalidArgument):
        sp.generate_matrix(sp.GridSpec(0, 1, 1))
    with pytest.raises(sp.InvalidArgument):
        sp.generate_matrix(sp.GridSpec(100000, 100000, 100000))
    with pytest.raises(sp.TableOverflowError):
        sp.compress_values(sp.stencil_from_rows(300, [[(i, float(i + 1))] for i in range(300)]))
    assert sp.compress_values(sp.stencil_from_rows(300, [[(i, float(i + 1))] for i in range(300)]),
                              value_table_limit=300).info.m == 300


def test_validate_catches_corruption(sp, orc):
    ref = orc.generate_matrix(3, 3, 3)
    vt = orc.compress_values(ref)
    ends = vt.ends.copy()
    ends[1] = 0  # non-monotone
    bad = sp.upload_vt(vt.n, vt.width, vt.table, vt.sorted_columns, ends)
    with pytest.raises(sp.IntegrityError):
        sp.validate(bad)
    with pytest.raises(sp.IntegrityError):
        sp.decompress(bad)
    pc = orc.compress_patterns(ref)
    ids = pc.row_pattern.copy()
    ids[0] = 13  # interior pattern on a corner row -> column out of range
    bad = sp.upload_pattern(pc.n, pc.table, pc.disp_offsets, pc.disp_flat, pc.ends_flat, ids)
    with pytest.raises(sp.IntegrityError):
        sp.validate(bad)
    sp.validate(sp.upload_pattern(pc.n, pc.table, pc.disp_offsets, pc.disp_flat, pc.ends_flat, pc.row_pattern))


def test_128_cubed_streams_against_oracle(sp, orc):
    """BASELINE configs[1] size: device-built compressed streams equal the oracle's byte for byte."""
    g = (128, 128, 128)
    m = sp.generate_matrix(sp.GridSpec(*g))
    assert m.nnz == (3 * 128 - 2) ** 3
    pc = sp.compress_patterns(m, True)
    ref = orc.compress_patterns_grid(*g, values_in_pattern=True)
    assert_pattern(pc, ref)
    chunk = orc.generate_matrix(*g, row_begin=1000000, row_end=1100000)
    rs = m.download("row_start", 1000000, 100001)
    assert same(rs - rs[0], chunk.row_start)
    assert same(m.download("cols", int(rs[0]), chunk.nnz), chunk.cols)


def test_config4_128_cubed(sp, orc):
    """BASELINE configs[3]: 128^3 with 10% perturbed rows -> hybrid format with exception rows."""
    g = (128, 128, 128)
    m = sp.generate_matrix(sp.GridSpec(*g), perturb=PERT)
    pc = sp.compress_patterns(m, True, min_pattern_rows=2)
    ref = orc.compress_patterns_grid(*g, perturb=PERT, values_in_pattern=True, min_pattern_rows=2)
    assert_pattern(pc, ref)
    assert abs(ref.n_exc / ref.n - 0.1) < 0.005 and 27 <= ref.w_exc <= 31
    n = ref.n
    x = orc.make_test_vector(n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    y_ref = np.empty(n)
    orc.spmv_rows(ref, x, y_ref, 0, n, threads=8)
    assert same(sp.spmv(pc, x), y_ref)
    # against the uncompressed ELL of the same matrix: 1e-12 relative per row
    ell = sp.to_ell(m)
    dx = sp.DeviceVector.from_host(x)
    dy1, dy2, sc = sp.DeviceVector(n), sp.DeviceVector(n), sp.DeviceVector(n)
    sp.spmv_rows(ell, dx, dy1, 0, n)
    sp.spmv_rows(pc, dx, dy2, 0, n)
    sp.row_abs_scale(m, dx, sc)
    worst, _ = sp.compare(dy2, dy1, n, scale=sc)
    assert worst <= 1e-12


def test_config5_512_cubed_single_gpu(sp):
    """BASELINE configs[4] on one GPU (it fits: CSR 44 GB build-time, 0.54 GB of ids resident): the matrix is
    generated and compressed on the device (n*27 > 2^31, so 64-bit slot offsets are exercised) and checked
    through size-independent properties."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < 120e9:
        pytest.skip("needs ~100 GB of free device memory")
    g = (512, 512, 512)
    n = 512 ** 3
    m = sp.generate_matrix(sp.GridSpec(*g))
    assert m.n == n and m.nnz == (3 * 512 - 2) ** 3  # nnz formula, SURVEY section 8
    pc = sp.compress_patterns(m, True)
    info = pc.info
    assert (info.n_patterns, info.n_exc, info.kernel_plan) == (27, 0, 1)
    assert (info.box_stride_y, info.box_stride_z) == (512, 512 * 512)
    ids = pc.download("row_pattern").reshape(512, 512, 512)
    assert len(np.unique(ids[1:-1, 1:-1, 1:-1])) == 1 and int(ids[1, 1, 1]) == 13  # interior rows share one id
    del ids, m
    # A*ones: interior exactly 0, everything >= 0; A*x agrees between the box and the List-1 kernels
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    sp.spmv_rows(pc, x, y, 0, n)
    yv = y.view(512, 512, 512)
    assert bool((yv[1:-1, 1:-1, 1:-1] == 0).all()) and bool((y >= 0).all())
    assert float(yv[0, 0, 0]) == 19.0 and float(yv[0, 0, 1]) == 15.0  # corner 26-7, edge 26-11
    sp.check(sp.lib.spmvb_vec_fill(x.data_ptr(), n, sp.RANDOM, 7, -1.0, 1.0, 0, None))
    y2 = torch.empty(n, dtype=torch.float64, device="cuda")
    sp.spmv_rows(pc, x, y, 0, n)
    sp.set_option("pattern_kernel", 1)
    try:
        sp.spmv_rows(pc, x, y2, 0, n)
    finally:
        sp.set_option("pattern_kernel", 0)
    assert sp.compare(y, y2, n) == (0.0, 0)
    # linearity within 1e-12: A(2x) == 2 A x exactly (power of two), partition invariance (kernels.hpp:27-29)
    x.mul_(2.0)
    sp.spmv_rows(pc, x, y2, 0, n // 2 + 12345)
    sp.spmv_rows(pc, x, y2, n // 2 + 12345, n)
    assert bool(torch.equal(y2, y * 2.0))
