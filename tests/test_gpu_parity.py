"""GPU parity tests: the CUDA SpMV path, called through the C-ABI, against the CPU
oracle on identical seeded inputs.  Integer / index streams and y are compared
bit-for-bit (the summation order of each format is kept, so y is bit-exact)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRIDS = [(1, 1, 1), (2, 2, 2), (3, 3, 3), (4, 4, 4), (5, 4, 3), (2, 5, 1), (7, 1, 4), (8, 3, 2), (6, 6, 6),
         (33, 9, 5), (40, 37, 11), (32, 32, 32), (100, 7, 9)]


@pytest.fixture(scope="module")
def sp():
    import paper_1612_00530_b200 as sp
    assert sp.device_count() >= 1
    return sp


def up_ell(sp, e):
    return sp.upload_ell(e.n, e.width, e.nnz, e.values, e.columns, row_offset=e.row_offset)


def up_vt(sp, v):
    return sp.upload_vt(v.n, v.width, v.table, v.sorted_columns, v.ends, row_offset=v.row_offset)


def up_pat(sp, p, row_offset=0):
    return sp.upload_pattern(p.n, p.table, p.disp_offsets, p.disp_flat, p.ends_flat, p.row_pattern,
                             p.values_in_pattern, p.exc_rows, p.exc_values, p.exc_columns, p.w_exc,
                             row_offset=row_offset)


def run(sp, a, x, begin=0, end=None, x_col0=0, n_rows=None):
    n = a.n if n_rows is None else n_rows
    dx = sp.DeviceVector.from_host(x)
    dy = sp.DeviceVector.from_host(np.full(n, np.nan))
    sp.spmv_rows(a, dx, dy, begin, n if end is None else end, x_col0=x_col0)
    return dy.to_host()


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("g", GRIDS)
def test_all_formats_bit_exact(sp, orc, g):
    m = orc.generate_matrix(*g)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    ell, vt, pc = orc.to_ell(m), orc.compress_values(m), orc.compress_patterns(m, False)
    d_ell, d_vt, d_pc = up_ell(sp, ell), up_vt(sp, vt), up_pat(sp, pc)
    # uploaded streams come back byte for byte
    assert d_ell.download("values").tobytes() == ell.values.tobytes()
    assert d_ell.download("columns").tobytes() == ell.columns.tobytes()
    assert d_vt.download("sorted_columns").tobytes() == vt.sorted_columns.tobytes()
    assert d_vt.download("ends").tobytes() == vt.ends.tobytes()
    assert d_pc.download("row_pattern").tobytes() == pc.row_pattern.tobytes()
    assert d_pc.download("disp_flat").tobytes() == pc.disp_flat.tobytes()
    for dev, ref in ((d_ell, ell), (d_vt, vt), (d_pc, pc)):
        y = run(sp, dev, x)
        assert np.array_equal(bits(y), bits(orc.spmv(ref, x))), f"format {dev.format} grid {g}"
        assert np.array_equal(bits(sp.spmv(dev, x)), bits(y))  # host-buffer entry point
    assert d_pc.info.nnz == m.nnz and d_vt.info.nnz == m.nnz
    # cross-format agreement 1e-13 relative per row, scale = sum |a_ik x_k|
    scale = orc.row_abs_scale(m, x)
    ys = [run(sp, d, x) for d in (d_ell, d_vt, d_pc)]
    for y in ys[1:]:
        assert (np.abs(y - ys[0]) / scale).max() <= 1e-13


@pytest.mark.parametrize("g", [(4, 4, 4), (6, 6, 6), (33, 9, 5), (40, 37, 11), (32, 32, 32), (128, 20, 12), (64, 33, 9),
                               (192, 17, 10), (100, 18, 11)])
@pytest.mark.parametrize("kernel", [1, 2, 3])
def test_pattern_kernels_generic_and_box(sp, orc, g, kernel):
    m = orc.generate_matrix(*g)
    pc = orc.compress_patterns(m, True)
    d = up_pat(sp, pc)
    info = d.info
    assert info.kernel_plan == 1 and (info.box_stride_y, info.box_stride_z) == (g[0], g[0] * g[1])
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=3, lo=-1.0, hi=1.0)
    sp.set_option("pattern_kernel", kernel)
    try:
        y = run(sp, d, x)
    finally:
        sp.set_option("pattern_kernel", 0)
    assert np.array_equal(bits(y), bits(orc.spmv(pc, x)))


@pytest.mark.parametrize("march", [1, 5, 11, 12, 20, 30, 35, 47, 62, 70])
@pytest.mark.parametrize("g", [(40, 37, 11), (128, 36, 20), (192, 40, 19), (256, 20, 12), (264, 18, 11), (512, 19, 15)])
def test_box_march_variants(sp, orc, march, g):
    if not sp.get_option("lab_build"):
        # the measured alternatives exist only in libspmvcomp_b200_lab.so (make LAB=1; SPMVB_LIB selects it)
        with pytest.raises(sp.InvalidArgument):
            sp.set_option("box_march", march)
        pytest.skip("lab variants are not part of the default library")
    m = orc.generate_matrix(*g)
    pc = orc.compress_patterns(m, True)
    d = up_pat(sp, pc)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=5, lo=-1.0, hi=1.0)
    sp.set_option("box_march", march)
    try:
        y = run(sp, d, x)
    finally:
        sp.set_option("box_march", 0)
    assert np.array_equal(bits(y), bits(orc.spmv(pc, x)))


def test_no_box_plan_for_flat_grids(sp, orc):
    for g in [(2, 2, 2), (7, 1, 4), (3, 3, 1)]:
        d = up_pat(sp, orc.compress_patterns(orc.generate_matrix(*g)))
        assert d.info.kernel_plan == 0
    with pytest.raises(sp.InvalidArgument):
        sp.set_option("pattern_kernel", 2)
        try:
            d = up_pat(sp, orc.compress_patterns(orc.generate_matrix(2, 2, 2)))
            run(sp, d, np.ones(8))
        finally:
            sp.set_option("pattern_kernel", 0)


@pytest.mark.parametrize("vals", [(26.0, -1.0), (-4.0, 1.5), (2.0, 2.0), (0.5, 3.0)])
def test_value_pairs_and_centre_position(sp, orc, vals):
    """centre last (off < diag), centre first (off > diag), single-value table, generic multiply."""
    diag, off = vals
    test_value_pairs_big(sp, orc, vals)
    m = orc.generate_matrix(9, 8, 7, diag, off)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=11, lo=-1.0, hi=1.0)
    for ref, dev in ((orc.to_ell(m), None), (orc.compress_values(m), None), (orc.compress_patterns(m), None)):
        dev = {orc.Ell: up_ell, orc.Vt: up_vt, orc.Pattern: up_pat}[type(ref)](sp, ref)
        assert np.array_equal(bits(run(sp, dev, x)), bits(orc.spmv(ref, x)))


def test_value_pairs_big(sp, orc, vals=(0.5, 3.0)):
    """Same on a grid wide enough for the guard-free vector march."""
    diag, off = vals
    m = orc.generate_matrix(128, 20, 12, diag, off)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=11, lo=-1.0, hi=1.0)
    ref = orc.compress_patterns(m)
    assert np.array_equal(bits(run(sp, up_pat(sp, ref), x)), bits(orc.spmv(ref, x)))


def test_row_ranges_big_grid(sp, orc):
    """Ragged row ranges on a grid with interior tiles: every partition gives the single-call result."""
    m = orc.generate_matrix(128, 20, 12)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    ref = orc.compress_patterns(m)
    dev = up_pat(sp, ref)
    full = orc.spmv(ref, x)
    dx = sp.DeviceVector.from_host(x)
    dy = sp.DeviceVector.from_host(np.full(m.n, np.nan))
    plane = 128 * 20
    cuts = [0, 2, 2 * plane, 2 * plane + 130, 5 * plane + 7, 9 * plane, m.n]
    for b, e in zip(cuts[:-1], cuts[1:]):
        sp.spmv_rows(dev, dx, dy, b, e)
    assert np.array_equal(bits(dy.to_host()), bits(full))


def test_row_ranges_untouched_and_bit_identical(sp, orc):
    """kernels.hpp:27-29: partitions give the single-call result; other rows are not written."""
    m = orc.generate_matrix(20, 13, 9)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    for ref, up in ((orc.to_ell(m), up_ell), (orc.compress_values(m), up_vt), (orc.compress_patterns(m), up_pat)):
        dev = up(sp, ref)
        full = orc.spmv(ref, x)
        dx = sp.DeviceVector.from_host(x)
        dy = sp.DeviceVector.from_host(np.full(m.n, 123.0))
        cuts = [0, 1, 130, 131, 777, 1500, m.n]
        for b, e in zip(cuts[:-1], cuts[1:]):
            if (b, e) == (131, 777):
                continue  # leave a hole
            sp.spmv_rows(dev, dx, dy, b, e)
        y = dy.to_host()
        assert np.all(y[131:777] == 123.0)
        keep = np.r_[0:131, 777:m.n]
        assert np.array_equal(bits(y[keep]), bits(full[keep]))
        with pytest.raises(sp.InvalidArgument):
            sp.spmv_rows(dev, dx, dy, 0, m.n + 1)
        with pytest.raises(sp.InvalidArgument):  # length mismatch
            sp.spmv(dev, np.ones(m.n - 1))


@pytest.mark.parametrize("g", [(12, 10, 9), (128, 18, 9)])
def test_slab_with_ghost_planes(sp, orc, g):
    """z-slab: local ids/ELL slices with global columns, ghosted local x (x_col0 = first ghost column)."""
    nx, ny, nz = g
    plane = nx * ny
    m = orc.generate_matrix(nx, ny, nz)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    pc, ell, vt = orc.compress_patterns(m, True), orc.to_ell(m), orc.compress_values(m)
    full = {k: orc.spmv(f, x) for k, f in (("p", pc), ("e", ell), ("v", vt))}
    for z0, z1 in ((0, 3), (3, 7), (7, 9)):
        r0, r1 = z0 * plane, z1 * plane
        g0, g1 = max(z0 - 1, 0) * plane, min(z1 + 1, nz) * plane  # ghosted column range
        xl = x[g0:g1]
        nl = r1 - r0
        w = ell.width
        d_p = sp.upload_pattern(nl, pc.table, pc.disp_offsets, pc.disp_flat, pc.ends_flat, pc.row_pattern[r0:r1],
                                True, row_offset=r0)
        d_e = sp.upload_ell(nl, w, 0, ell.values[r0 * w:r1 * w], ell.columns[r0 * w:r1 * w], row_offset=r0)
        d_v = sp.upload_vt(nl, w, vt.table, vt.sorted_columns[r0 * w:r1 * w], vt.ends[r0 * 2:r1 * 2], row_offset=r0)
        for key, dev in (("p", d_p), ("e", d_e), ("v", d_v)):
            y = run(sp, dev, xl, x_col0=g0)
            assert np.array_equal(bits(y), bits(full[key][r0:r1])), (key, z0, z1)


@pytest.mark.parametrize("g", [(16, 16, 16), (48, 40, 36), (128, 20, 12)])
def test_hybrid_exception_rows(sp, orc, g):
    """Config-4 style matrix: perturbed rows become uncompressed exception rows."""
    m = orc.generate_matrix(*g, perturb=(11, 0.1, 0.1))
    pc = orc.compress_patterns(m, True, min_pattern_rows=2)
    assert pc.n_exc > 0 and abs(pc.n_exc / m.n - 0.1) < 0.03
    orc.validate(pc)
    assert orc.decompress(pc) == m
    d = up_pat(sp, pc)
    assert d.info.nnz == m.nnz
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    ref = orc.spmv(pc, x)
    exc = pc.exc_rows  # exception rows are summed in ELL slot order == ascending-column (CSR) order
    assert np.array_equal(bits(ref[exc]), bits(orc.spmv(m, x)[exc]))
    for kernel in (1, 2, 3):
        sp.set_option("pattern_kernel", kernel)
        try:
            y = run(sp, d, x)
        finally:
            sp.set_option("pattern_kernel", 0)
        assert np.array_equal(bits(y), bits(ref))
    # the exception block from shared-memory windows of x (csrc/spmv_exception.cu), whole and over ragged row ranges
    dx = sp.DeviceVector.from_host(x)
    for ek in (64, 32):
        sp.set_option("exception_kernel", ek)
        try:
            assert np.array_equal(bits(run(sp, d, x)), bits(ref))
            n = m.n
            for b, e in ((0, n // 3 + 1), (n // 3 + 1, n - 5), (n - 5, n), (7, 8)):
                dy = sp.DeviceVector.from_host(np.full(n, np.nan))
                sp.spmv_rows(d, dx, dy, b, e)
                yh = dy.to_host()
                assert np.array_equal(bits(yh[b:e]), bits(ref[b:e])) and np.all(np.isnan(yh[:b])) and np.all(np.isnan(yh[e:]))
        finally:
            sp.set_option("exception_kernel", 0)
    # the uncompressed ELL of the same matrix agrees to 1e-12 per row
    ell = orc.to_ell(m)
    y_ell = run(sp, up_ell(sp, ell), x)
    assert np.array_equal(bits(y_ell), bits(orc.spmv(ell, x)))
    assert (np.abs(y_ell - ref) / orc.row_abs_scale(m, x)).max() <= 1e-12


@pytest.mark.parametrize("ell_kernel", [0, 1, 2, 3])
def test_ell_vt_kernel_variants(sp, orc, ell_kernel):
    """TMA bulk pipeline (0), naive (1) and staged vector-load (2) kernels agree bit for bit with the oracle."""
    for g in [(5, 4, 3), (33, 9, 5), (64, 33, 9), (128, 20, 12)]:
        m = orc.generate_matrix(*g)
        x = orc.make_test_vector(m.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
        ell, vt = orc.to_ell(m), orc.compress_values(m)
        sp.set_option("ell_kernel", ell_kernel)
        try:
            ye, yv = run(sp, up_ell(sp, ell), x), run(sp, up_vt(sp, vt), x)
            dx = sp.DeviceVector.from_host(x)
            dy = sp.DeviceVector.from_host(np.full(m.n, 5.0))
            sp.spmv_rows(up_ell(sp, ell), dx, dy, 3, m.n - 2)  # ragged range
            part = dy.to_host()
        finally:
            sp.set_option("ell_kernel", 0)
        assert np.array_equal(bits(ye), bits(orc.spmv(ell, x))) and np.array_equal(bits(yv), bits(orc.spmv(vt, x)))
        assert np.all(part[:3] == 5.0) and np.all(part[-2:] == 5.0)
        assert np.array_equal(bits(part[3:-2]), bits(orc.spmv(ell, x)[3:-2]))


def test_fig_row_and_explicit_rows(sp, orc):
    rows = [[(i, 26.0)] for i in range(66)]
    rows[50] = [(45, -1.0), (49, -1.0), (50, 26.0), (51, -1.0), (65, -1.0)]
    m = orc.stencil_from_rows(66, rows)
    x = np.ones(66)
    for ref, up in ((orc.to_ell(m), up_ell), (orc.compress_values(m), up_vt), (orc.compress_patterns(m), up_pat)):
        assert run(sp, up(sp, ref), x)[50] == 22.0


def test_vector_fill_matches_oracle(sp, orc):
    n = 100003
    for kind, kw in ((orc.ONES, {}), (orc.LINEAR, {}), (orc.RANDOM, dict(seed=7)),
                     (orc.RANDOM, dict(seed=7, lo=-1.0, hi=1.0)), (orc.RANDOM, dict(seed=9, lo=-0.1, hi=0.1))):
        dev = sp.make_test_vector(n, kind, first_index=17, **kw).to_host()
        ref = orc.make_test_vector(n, kind, first_index=17, **kw)
        assert np.array_equal(bits(dev), bits(ref))
    with pytest.raises(sp.InvalidArgument):
        sp.make_test_vector(4, sp.RANDOM)


def test_compare_helper(sp):
    a = np.array([1.0, 2.0, 0.0, 4.0])
    b = np.array([1.0, 2.0 + 4e-16, 0.0, 4.0])
    da, db = sp.DeviceVector.from_host(a), sp.DeviceVector.from_host(b)
    worst, bad = sp.compare(da, db, 4)
    assert bad == 1 and 0 < worst < 1e-15
    assert sp.compare(da, da, 4) == (0.0, 0)


def test_pattern_upload_integrity(sp, orc):
    pc = orc.compress_patterns(orc.generate_matrix(3, 3, 3))
    ids = pc.row_pattern.copy()
    ids[3] = 99
    with pytest.raises(sp.IntegrityError):
        sp.upload_pattern(pc.n, pc.table, pc.disp_offsets, pc.disp_flat, pc.ends_flat, ids)
    ends = pc.ends_flat.copy()
    ends[1] = 0
    with pytest.raises(sp.IntegrityError):
        sp.upload_pattern(pc.n, pc.table, pc.disp_offsets, pc.disp_flat, ends, pc.row_pattern)


def test_128_cubed_properties(sp, orc):
    """BASELINE config 2 size: compressed vs uncompressed on the GPU, plus a sampled oracle check."""
    g = (128, 128, 128)
    pc = orc.compress_patterns_grid(*g, values_in_pattern=True)
    d = up_pat(sp, pc)
    n = pc.n
    x = orc.make_test_vector(n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    y = run(sp, d, x)
    ref = np.empty(n)
    orc.spmv_rows(pc, x, ref, 0, n, threads=8)
    assert np.array_equal(bits(y), bits(ref))
    sp.set_option("pattern_kernel", 1)
    try:
        assert np.array_equal(bits(run(sp, d, x)), bits(ref))
    finally:
        sp.set_option("pattern_kernel", 0)
    # A*ones: interior exactly 0, everything >= 0
    y1 = run(sp, d, np.ones(n)).reshape(g[::-1])
    assert np.all(y1[1:-1, 1:-1, 1:-1] == 0.0) and np.all(y1 >= 0.0)


def test_acceptance_5_random_small_grids_against_the_dense_product(sp):
    """SPEC.md:515 on the device path: 25 randomized grids <= 6^3 with seeded vectors, built and multiplied on the GPU;
    vt and pattern match the dense brute-force product and the ELL backend within 1e-13 element-wise relative."""
    from tests.dense_ref import dense_stencil, rel_err
    rng = np.random.default_rng(515)
    for trial in range(25):
        g = tuple(int(v) for v in rng.integers(1, 7, size=3))
        n = g[0] * g[1] * g[2]
        x = rng.uniform(-1.0, 1.0, size=n)
        a = dense_stencil(*g)
        ref = a @ x
        scale = np.abs(a) @ np.abs(x)
        m = sp.generate_matrix(sp.GridSpec(*g))
        ys = {"ell": sp.spmv(sp.to_ell(m), x), "vt": sp.spmv(sp.compress_values(m), x),
              "pattern": sp.spmv(sp.compress_patterns(m, False), x), "pattern-values": sp.spmv(sp.compress_patterns(m, True), x)}
        for name, y in ys.items():
            assert rel_err(y, ref, scale).max() <= 1e-13, (g, name)
            assert rel_err(y, ys["ell"], scale).max() <= 1e-13, (g, name)
