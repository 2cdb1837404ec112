"""Tensor-ring pattern kernel (csrc/spmv_pattern_tma.cu): bit-exact against the oracle's List 1
 on aligned and misaligned views, ragged ranges, slabs and hybrid matrices."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from tests.test_gpu_parity import bits, run, sp, up_pat  # noqa: E402,F401

# default schedule, chunk per warp, ids by loads, round-robin tiles (per CTA, per warp), 4 planes/thread, two lines per step (chunks, tiles)
RING = [90, 101, 107, 108, 109, 110, 111, 112]


def ring_run(sp, d, x, march, lines=0, must_ring=True, **kw):
    sp.set_option("box_march", march)
    sp.set_option("box_lines", lines)
    try:
        y = run(sp, d, x, **kw)
        used = sp.get_option("last_pattern_kernel")
    finally:
        sp.set_option("box_march", 0)
        sp.set_option("box_lines", 0)
    if must_ring:
        assert used == 9, f"tensor-ring kernel not used (kernel family {used})"
    return y


@pytest.mark.parametrize("march", RING)
@pytest.mark.parametrize("g", [(68, 10, 9), (100, 18, 11), (130, 9, 8), (128, 36, 20), (192, 40, 19), (256, 20, 12), (264, 18, 11),
                               (512, 19, 15)])
def test_ring_variants_bit_exact(sp, orc, march, g):
    m = orc.generate_matrix(*g)
    pc = orc.compress_patterns(m, True)
    d = up_pat(sp, pc)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=5, lo=-1.0, hi=1.0)
    assert np.array_equal(bits(ring_run(sp, d, x, march)), bits(orc.spmv(pc, x)))


@pytest.mark.parametrize("lines", [1, 2, 3, 7, 64])
def test_ring_march_lengths(sp, orc, lines):
    m = orc.generate_matrix(128, 21, 10)
    pc = orc.compress_patterns(m, True)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=6, lo=-1.0, hi=1.0)
    assert np.array_equal(bits(ring_run(sp, up_pat(sp, pc), x, 90, lines)), bits(orc.spmv(pc, x)))


@pytest.mark.parametrize("leftover", [0, 1, 2])
@pytest.mark.parametrize("march,lines", [(90, 0), (90, 100), (90, 47), (108, 16), (108, 40), (110, 0), (111, 0), (111, 5), (111, 28), (111, 60),
                                         (112, 0), (112, 7), (112, 16), (112, 40)])
def test_ring_leftover_column_schemes(sp, orc, leftover, march, lines):
    """64 | nx: column nx-1 lies past the last strip.  Chunk-per-CTA kernels gather its operands per line and sum its rows
    after the march (marches longer than the side buffer are split; tiles longer than it keep the per-step sums); option
    ring_leftover = 2 forces the per-step sums, 1 the row-by-row tail.  Every scheme is the oracle's List 1 bit for bit."""
    m = orc.generate_matrix(256, 100, 9)
    pc = orc.compress_patterns(m, True)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=8, lo=-1.0, hi=1.0)
    sp.set_option("ring_leftover", leftover)
    try:
        y = ring_run(sp, up_pat(sp, pc), x, march, lines)
    finally:
        sp.set_option("ring_leftover", 0)
    assert np.array_equal(bits(y), bits(orc.spmv(pc, x)))


@pytest.mark.parametrize("march", [90, 108, 111, 112])
def test_ring_ragged_ranges(sp, orc, march):
    """Partitions at arbitrary (even and odd) rows give the single-call result; other rows stay untouched."""
    m = orc.generate_matrix(128, 20, 12)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    ref = orc.compress_patterns(m)
    dev = up_pat(sp, ref)
    full = orc.spmv(ref, x)
    dx = sp.DeviceVector.from_host(x)
    dy = sp.DeviceVector.from_host(np.full(m.n, 123.0))
    plane = 128 * 20
    cuts = [0, 2, 131, 2 * plane, 2 * plane + 130, 5 * plane + 7, 9 * plane, m.n - 1, m.n]
    sp.set_option("box_march", march)
    try:
        for b, e in zip(cuts[:-1], cuts[1:]):
            if (b, e) == (2 * plane + 130, 5 * plane + 7):
                continue  # leave a hole
            sp.spmv_rows(dev, dx, dy, b, e)
            assert sp.get_option("last_pattern_kernel") == 9
    finally:
        sp.set_option("box_march", 0)
    y = dy.to_host()
    hole = slice(2 * plane + 130, 5 * plane + 7)
    assert np.all(y[hole] == 123.0)
    keep = np.r_[0:hole.start, hole.stop:m.n]
    assert np.array_equal(bits(y[keep]), bits(full[keep]))


@pytest.mark.parametrize("g", [(128, 18, 9), (70, 12, 10)])
def test_ring_slab_with_ghost_planes(sp, orc, g):
    nx, ny, nz = g
    plane = nx * ny
    m = orc.generate_matrix(nx, ny, nz)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    pc = orc.compress_patterns(m, True)
    full = orc.spmv(pc, x)
    for z0, z1 in ((0, 3), (3, 7), (7, nz)):
        r0, r1 = z0 * plane, z1 * plane
        g0, g1 = max(z0 - 1, 0) * plane, min(z1 + 1, nz) * plane
        d_p = sp.upload_pattern(r1 - r0, pc.table, pc.disp_offsets, pc.disp_flat, pc.ends_flat, pc.row_pattern[r0:r1],
                                True, row_offset=r0)
        y = ring_run(sp, d_p, x[g0:g1], 90, x_col0=g0)
        assert np.array_equal(bits(y), bits(full[r0:r1])), (z0, z1)


@pytest.mark.parametrize("nx", [128, 256])  # 256: strips in fours -> 6 planes/thread, ids by per-thread loads
def test_ring_misaligned_view_falls_back_per_row(sp, orc, nx):
    """x_col0 that is not a multiple of the plane: the zero-filled view disagrees with the masks of the
    rows on the view's faces, which must then be recomputed by List 1 -- same bits."""
    ny, nz = 10, 9
    plane = nx * ny
    m = orc.generate_matrix(nx, ny, nz)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=8, lo=-1.0, hi=1.0)
    pc = orc.compress_patterns(m, True)
    full = orc.spmv(pc, x)
    r0, r1 = 3 * plane, 6 * plane
    for g0 in (2 * plane - 2 * nx - 6, 2 * plane - nx - 2, 2 * plane - 2):  # even offsets, not plane / line aligned
        d_p = sp.upload_pattern(r1 - r0, pc.table, pc.disp_offsets, pc.disp_flat, pc.ends_flat, pc.row_pattern[r0:r1],
                                True, row_offset=r0)
        for march in (90, 111, 112):
            y = ring_run(sp, d_p, x[g0:7 * plane], march, x_col0=g0)
            assert np.array_equal(bits(y), bits(full[r0:r1])), (g0, march)


@pytest.mark.parametrize("g", [(128, 20, 12), (96, 40, 36)])
def test_ring_hybrid_exception_rows(sp, orc, g):
    m = orc.generate_matrix(*g, perturb=(11, 0.1, 0.1))
    pc = orc.compress_patterns(m, True, min_pattern_rows=2)
    assert pc.n_exc > 0
    d = up_pat(sp, pc)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    for march in (90, 111, 112):
        assert np.array_equal(bits(ring_run(sp, d, x, march)), bits(orc.spmv(pc, x))), march


def test_ring_nonfinite_neighbours_do_not_leak(sp, orc):
    """Absent entries are never read as operands: NaN in x reaches exactly the rows that reference it."""
    m = orc.generate_matrix(128, 12, 10)
    pc = orc.compress_patterns(m, True)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=9, lo=-1.0, hi=1.0)
    x[127] = np.nan  # last column of line 0: not a neighbour of row 128 (column 0 of line 1)
    ref = orc.spmv(pc, x)
    ok = ~np.isnan(ref)
    for march in (90, 111):
        y = ring_run(sp, up_pat(sp, pc), x, march)
        assert np.array_equal(np.isnan(y), np.isnan(ref)) and np.array_equal(bits(y[ok]), bits(ref[ok]))
        assert np.isnan(y[126]) and not np.isnan(y[128])


@pytest.mark.parametrize("vals", [(26.0, -1.0), (-4.0, 1.5), (2.0, 2.0), (0.5, 3.0), (-1.0, -1.0), (-3.0, -1.0)])
def test_ring_value_pairs_and_centre_position(sp, orc, vals):
    """centre last / first / in place, off-diagonal -1 and general: the default variant serves them all."""
    diag, off = vals
    m = orc.generate_matrix(128, 11, 10, diag, off)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=11, lo=-1.0, hi=1.0)
    ref = orc.compress_patterns(m)
    for march in (0, 111, 112):  # (the two-lines step has its own general instantiation)
        assert np.array_equal(bits(ring_run(sp, up_pat(sp, ref), x, march)), bits(orc.spmv(ref, x))), march


def test_ring_is_the_default_for_large_ranges(sp, orc):
    m = orc.generate_matrix(128, 12, 10)
    pc = orc.compress_patterns(m, True)
    d = up_pat(sp, pc)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=5, lo=-1.0, hi=1.0)
    y = run(sp, d, x)
    assert sp.get_option("last_pattern_kernel") == 9
    assert np.array_equal(bits(y), bits(orc.spmv(pc, x)))
    dx, dy = sp.DeviceVector.from_host(x), sp.DeviceVector.from_host(np.zeros(m.n))
    sp.spmv_rows(d, dx, dy, 0, 3 * 128 * 12)  # a few planes, few rows: List 1 with a thread per row (one round of gathers)
    assert sp.get_option("last_pattern_kernel") == 1
    assert np.array_equal(bits(dy.to_host()[:3 * 128 * 12]), bits(orc.spmv(pc, x)[:3 * 128 * 12]))
    sp.set_option("box_march", 3)  # the sliding-window kernel, forced
    try:
        sp.spmv_rows(d, dx, dy, 0, 3 * 128 * 12)
        assert sp.get_option("last_pattern_kernel") == 3
    finally:
        sp.set_option("box_march", 0)
    assert np.array_equal(bits(dy.to_host()[:3 * 128 * 12]), bits(orc.spmv(pc, x)[:3 * 128 * 12]))


@pytest.mark.parametrize("march", [0, 101, 109, 111, 112])
def test_ring_ghost_planes_beyond_the_grid_faces(sp, orc, march):
    """x padded by one (unreferenced) plane at each end, x_col0 = -plane (the single-rank SlabLayout): the rows
    of the first and last grid plane are sub-boxes whose missing entries are inside the view."""
    nx, ny, nz = 128, 12, 10
    plane = nx * ny
    m = orc.generate_matrix(nx, ny, nz)
    pc = orc.compress_patterns(m, True)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=12, lo=-1.0, hi=1.0)
    xg = np.concatenate([np.full(plane, np.nan), x, np.full(plane, np.nan)])  # ghosts must never be read as operands
    y = ring_run(sp, up_pat(sp, pc), xg, march, x_col0=-plane, n_rows=m.n)
    assert np.array_equal(bits(y), bits(orc.spmv(pc, x)))


def test_ring_randomised_shapes_ranges_and_views(sp, orc):
    """Random grids (partial strips, one or two left-over columns, strips in fours, plane counts that are not a
    multiple of the planes per thread), row ranges cut anywhere and x views with and without ghost planes: the
    default dispatch (tensor ring where it applies) is bit-identical to List 1 on the CPU."""
    rng = np.random.default_rng(20260117)
    used_ring = 0
    for trial in range(36):
        nx = int(rng.choice([256, 512, 256, 68, 70, 126, 128, 130, 192, 194, 258, 320, 384]))
        ny = int(rng.integers(2, 9))
        nz = int(rng.integers(8, 23))
        m = orc.generate_matrix(nx, ny, nz)
        pc = orc.compress_patterns(m, True)
        n, plane = m.n, nx * ny
        x = orc.make_test_vector(n, orc.RANDOM, seed=100 + trial, lo=-1.0, hi=1.0)
        full = orc.spmv(pc, x)
        # a slab of planes [z0, z1) with ghost planes (or more) on either side, possibly beyond the grid faces
        z0 = int(rng.integers(0, 3))
        z1 = nz - int(rng.integers(0, 3))
        r0, r1 = z0 * plane, z1 * plane
        below, above = int(rng.integers(1, 3)), int(rng.integers(1, 3))
        g_lo, g_hi = (z0 - below) * plane, (z1 + above) * plane
        xl = np.full(g_hi - g_lo, np.nan)  # positions outside the grid are never referenced
        lo, hi = max(g_lo, 0), min(g_hi, n)
        xl[lo - g_lo:hi - g_lo] = x[lo:hi]
        d = sp.upload_pattern(r1 - r0, pc.table, pc.disp_offsets, pc.disp_flat, pc.ends_flat, pc.row_pattern[r0:r1], True,
                              row_offset=r0)
        nl = r1 - r0
        cuts = sorted({0, nl, *(int(v) for v in rng.integers(0, nl + 1, size=2))})
        dx = sp.DeviceVector.from_host(xl)
        for march in (0, 90, 111, 112):  # the default dispatch, and the tensor ring forced also for ranges of a few planes (+ two lines per step)
            dy = sp.DeviceVector.from_host(np.full(nl, np.nan))
            sp.set_option("box_march", march)
            try:
                for b, e in zip(cuts[:-1], cuts[1:]):
                    sp.spmv_rows(d, dx, dy, b, e, x_col0=g_lo)
                    used_ring += march == 90 and sp.get_option("last_pattern_kernel") == 9
            finally:
                sp.set_option("box_march", 0)
            y = dy.to_host()
            assert np.array_equal(bits(y), bits(full[r0:r1])), (trial, march, nx, ny, nz, z0, z1, below, above, cuts)
    assert used_ring >= 60
