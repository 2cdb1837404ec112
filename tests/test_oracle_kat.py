"""Pins the CPU oracle against every known-answer the reference states for the
SpMV path (SPEC.md worked examples and
acceptance criteria 1-7).  Runs on CPU."""
import itertools

import numpy as np
import pytest

from tests.dense_ref import dense_stencil, rel_err

FIG_ROW = [(45, -1.0), (49, -1.0), (50, 26.0), (51, -1.0), (65, -1.0)]


def fig_matrix(orc, n=66):
    """A matrix whose row 50 is the paper's figure row; every other row is a lone diagonal."""
    rows = [[(i, 26.0)] for i in range(n)]
    rows[50] = FIG_ROW
    return orc.stencil_from_rows(n, rows)


# ---- K1-K3, K15: generator -------------------------------
def test_k1_single_node(orc):
    m = orc.generate_matrix(1, 1, 1)
    assert m.n == 1 and m.nnz == 1
    assert m.cols.tolist() == [0] and m.vals.tolist() == [26.0]


def test_k2_2x2x2(orc):
    m = orc.generate_matrix(2, 2, 2)
    assert m.n == 8
    for i in range(8):
        c, v = m.row(i)
        assert len(c) == 8 and v.sum() == 19.0 and sorted(v.tolist()) == [-1.0] * 7 + [26.0]


def test_k3_interior_row_4x4x4(orc):
    m = orc.generate_matrix(4, 4, 4)
    i = 1 + 4 * (1 + 4 * 1)
    c, v = m.row(i)
    assert len(c) == 27 and v.sum() == 0.0


@pytest.mark.parametrize("g", [(1, 1, 1), (2, 2, 2), (3, 3, 3), (4, 4, 4), (5, 4, 3), (2, 5, 1), (6, 6, 6), (8, 3, 2)])
def test_k15_generator_properties(orc, g):
    nx, ny, nz = g
    m = orc.generate_matrix(*g)
    assert orc.is_symmetric(m)
    assert m.nnz == (3 * nx - 2) * (3 * ny - 2) * (3 * nz - 2)
    rs = m.row_start
    counts = np.diff(rs)
    assert (counts == 27).sum() == max(nx - 2, 0) * max(ny - 2, 0) * max(nz - 2, 0)
    for i in range(m.n):
        c, _ = m.row(i)
        assert np.all(np.diff(c) > 0)
    assert np.array_equal(m.dense(), dense_stencil(*g))
    y = orc.spmv(m, np.ones(m.n))
    assert np.all(y >= 0.0)


def test_grid_validation(orc):
    with pytest.raises(orc.InvalidArgument):
        orc.generate_matrix(0, 1, 1)
    with pytest.raises(orc.InvalidArgument):  # SPEC.md:444 sizing error
        orc.generate_matrix(100000, 100000, 100000)


def test_test_vectors(orc):
    assert orc.make_test_vector(3, orc.ONES).tolist() == [1, 1, 1]
    assert orc.make_test_vector(3, orc.LINEAR).tolist() == [0, 1, 2]
    a = orc.make_test_vector(4, orc.RANDOM, seed=7)
    b = orc.make_test_vector(4, orc.RANDOM, seed=7)
    assert np.array_equal(a, b) and np.all((a >= 0) & (a < 1))  # SPEC.md:66, stencil.hpp:56
    assert not np.array_equal(a, orc.make_test_vector(4, orc.RANDOM, seed=8))
    with pytest.raises(orc.InvalidArgument):
        orc.make_test_vector(4, orc.RANDOM)
    # counter-based: a slab of the vector equals the slice of the whole
    whole = orc.make_test_vector(100, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    part = orc.make_test_vector(30, orc.RANDOM, seed=7, lo=-1.0, hi=1.0, first_index=50)
    assert np.array_equal(whole[50:80], part) and whole.min() >= -1 and whole.max() < 1


# ---- K4: the paper's figure row ---------
def test_k4_figure_row(orc):
    m = fig_matrix(orc)
    ell = orc.to_ell(m)
    w = ell.width
    assert w == 5
    assert ell.values[50 * w:51 * w].tolist() == [-1, -1, 26, -1, -1]
    assert ell.columns[50 * w:51 * w].tolist() == [45, 49, 50, 51, 65]
    vt = orc.compress_values(m)
    assert vt.table.tolist() == [-1.0, 26.0]
    assert vt.sorted_columns[50 * w:51 * w].tolist() == [45, 49, 51, 65, 50]
    assert vt.ends[100:102].tolist() == [4, 5]
    pc = orc.compress_patterns(m, False)
    disp, ends = pc.pattern(pc.row_pattern[50])
    assert disp == [-5, -1, 1, 15, 0] and ends == [4, 5]
    x = np.ones(66)
    for fmt in (ell, vt, pc):
        assert orc.spmv(fmt, x)[50] == 22.0
    back = orc.decompress(pc)
    c, v = back.row(50)
    assert c.tolist() == [45, 49, 50, 51, 65] and v.tolist() == [-1, -1, 26, -1, -1]
    assert orc.decompress(vt) == m and back == m


# ---- K5/K6: pattern count and value table --------
@pytest.mark.parametrize("g", [(1, 1, 1), (2, 2, 2), (3, 3, 3), (4, 4, 4), (5, 4, 3), (2, 5, 1), (6, 6, 6), (8, 3, 2), (7, 1, 4)])
def test_k5_k6_pattern_count_and_table(orc, g):
    nx, ny, nz = g
    m = orc.generate_matrix(*g)
    pc = orc.compress_patterns(m, True)
    assert pc.n_patterns == min(nx, 3) * min(ny, 3) * min(nz, 3)
    assert pc.n_exc == 0
    if m.n >= 2:
        assert pc.table.tolist() == [-1.0, 26.0]
        assert orc.scan_value_table(m).tolist() == [-1.0, 26.0]
    # every pattern referenced, ids valid
    assert sorted(set(pc.row_pattern.tolist())) == list(range(pc.n_patterns))
    # interior rows share one id
    ids = pc.row_pattern.reshape(nz, ny, nx)
    if min(g) >= 3:
        assert len(set(ids[1:-1, 1:-1, 1:-1].ravel().tolist())) == 1


def test_pattern_id_numbering_first_occurrence(orc):
    """Unpinned choice (1): ids issued in order of first occurrence, ascending rows."""
    pc = orc.compress_patterns(orc.generate_matrix(4, 4, 4), False)
    ids = pc.row_pattern.tolist()
    assert ids[:8] == [0, 1, 1, 2, 3, 4, 4, 5]
    seen = []
    for i in ids:
        if i not in seen:
            seen.append(i)
    assert seen == list(range(27))
    assert ids[1 + 4 * (1 + 4)] == 13


def test_table_overflow(orc):
    rows = [[(i, float(i + 1))] for i in range(300)]
    m = orc.stencil_from_rows(300, rows)
    with pytest.raises(orc.TableOverflowError):
        orc.compress_values(m)
    with pytest.raises(orc.TableOverflowError):
        orc.compress_patterns(m)
    assert orc.compress_values(m, limit=300).m == 300


# ---- K7: ELL ---------------------------------------------
def test_k7_ell(orc):
    e = orc.to_ell(orc.generate_matrix(1, 1, 1))
    assert (e.width, e.values.tolist(), e.columns.tolist()) == (1, [26.0], [0])
    m = orc.generate_matrix(2, 2, 2)
    e = orc.to_ell(m)
    assert e.width == 8 and np.all(e.values != 0.0)
    m = orc.generate_matrix(4, 4, 4)
    e = orc.to_ell(m)
    assert e.width == 27 and e.nnz == m.nnz
    v = e.values.reshape(64, 27)
    c = e.columns.reshape(64, 27)
    k = np.diff(m.row_start)
    for i in range(64):  # trailing padding = (0.0, own row)
        assert np.all(v[i, k[i]:] == 0.0) and np.all(c[i, k[i]:] == i)
    assert orc.to_stencil(e) == m


# ---- K8-K10: SpMV worked examples ----------------
def test_k8_1x1(orc):
    m = orc.generate_matrix(1, 1, 1)
    assert orc.spmv(orc.to_ell(m), [2.0]).tolist() == [52.0]
    assert orc.spmv(orc.compress_values(m), [1.0]).tolist() == [26.0]
    assert orc.spmv(orc.compress_patterns(m, True), [-1.0]).tolist() == [-26.0]
    vt = orc.compress_values(m)
    assert (vt.table.tolist(), vt.sorted_columns.tolist(), vt.ends.tolist()) == ([26.0], [0], [1])


def test_k9_ones(orc):
    m = orc.generate_matrix(4, 4, 4)
    for fmt in (orc.to_ell(m), orc.compress_values(m), orc.compress_patterns(m, False)):
        y = orc.spmv(fmt, np.ones(64)).reshape(4, 4, 4)
        assert np.all(y[1:3, 1:3, 1:3] == 0.0) and np.all(y >= 0.0)
    m2 = orc.generate_matrix(2, 2, 2)
    assert orc.spmv(orc.compress_patterns(m2, False), np.ones(8)).tolist() == [19.0] * 8


def test_k10_linear_dense(orc):
    m = orc.generate_matrix(3, 3, 3)
    x = orc.make_test_vector(27, orc.LINEAR)
    ref = dense_stencil(3, 3, 3) @ x
    assert np.array_equal(orc.spmv(orc.to_ell(m), x), ref)  # small integers: exact


def test_length_mismatch(orc):
    m = orc.generate_matrix(3, 3, 3)
    for fmt in (orc.to_ell(m), orc.compress_values(m), orc.compress_patterns(m)):
        with pytest.raises(orc.InvalidArgument):
            orc.spmv(fmt, np.ones(5))


# ---- K11: cross-format and dense agreement ---------------
def test_k11_cross_format_all_grids(orc):
    worst = 0.0
    for g in itertools.product(range(1, 7), repeat=3):
        m = orc.generate_matrix(*g)
        dense = dense_stencil(*g) if m.n <= 64 else None
        fmts = (orc.to_ell(m), orc.compress_values(m), orc.compress_patterns(m, False))
        for seed in (1, 2, 3):
            x = orc.make_test_vector(m.n, orc.RANDOM, seed=seed, lo=-1.0, hi=1.0)
            ys = [orc.spmv(f, x) for f in fmts]
            ref = orc.spmv(m, x)
            scale = orc.row_abs_scale(m, x)
            assert np.array_equal(ys[0], ref)  # ELL order == CSR ascending order
            for y in ys[1:]:
                worst = max(worst, (np.abs(y - ref) / scale).max())
            if dense is not None:
                worst = max(worst, (np.abs(dense @ x - ref) / scale).max())
    assert worst <= 1e-13


def test_linearity_and_symmetry(orc):
    m = orc.generate_matrix(5, 4, 6)
    pc = orc.compress_patterns(m, False)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=1, lo=-1, hi=1)
    z = orc.make_test_vector(m.n, orc.RANDOM, seed=2, lo=-1, hi=1)
    a, b = 0.75, -1.5
    lhs = orc.spmv(pc, a * x + b * z)
    rhs = a * orc.spmv(pc, x) + b * orc.spmv(pc, z)
    assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()
    s1, s2 = orc.spmv(pc, x) @ z, x @ orc.spmv(pc, z)
    assert abs(s1 - s2) <= 1e-12 * abs(s1)


def test_row_range_partition_is_bit_identical(orc):
    """kernels.hpp:27-29: any partition of the rows gives the single-call result."""
    m = orc.generate_matrix(6, 5, 4)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=7, lo=-1, hi=1)
    for fmt in (orc.to_ell(m), orc.compress_values(m), orc.compress_patterns(m)):
        ref = orc.spmv(fmt, x)
        y = np.full(m.n, np.nan)
        for b, e in ((0, 17), (17, 18), (18, 90), (90, m.n)):
            orc.spmv_rows(fmt, x, y, b, e)
        assert np.array_equal(y, ref)
        y2 = np.full(m.n, np.nan)
        orc.spmv_rows(fmt, x, y2, 0, m.n, threads=5)
        assert np.array_equal(y2, ref)
        y3 = np.full(m.n, 123.0)
        orc.spmv_rows(fmt, x, y3, 10, 20)
        assert np.all(y3[:10] == 123.0) and np.all(y3[20:] == 123.0)  # rows outside untouched


# ---- K12: lossless round trip and determinism ------------
def test_k12_round_trip_all_grids(orc):
    for g in itertools.product(range(1, 9), repeat=3):  # nx, ny, nz in [1,8] (acceptance criterion 4 asks for [1,6])
        m = orc.generate_matrix(*g)
        vt = orc.compress_values(m)
        pc = orc.compress_patterns(m, False)
        orc.validate(vt)
        orc.validate(pc)
        assert orc.decompress(vt) == m and orc.decompress(pc) == m
        assert orc.to_stencil(orc.to_ell(m)) == m
    m = orc.generate_matrix(6, 5, 4)
    a, b = orc.compress_patterns(m, True), orc.compress_patterns(m, True)
    for f in ("row_pattern", "disp_flat", "ends_flat", "disp_offsets", "table"):
        assert getattr(a, f).tobytes() == getattr(b, f).tobytes()
    g = orc.compress_patterns_grid(6, 5, 4, values_in_pattern=True)
    for f in ("row_pattern", "disp_flat", "ends_flat", "disp_offsets", "table"):
        assert getattr(a, f).tobytes() == getattr(g, f).tobytes()


def test_integrity_errors(orc):
    m = orc.generate_matrix(3, 3, 3)
    vt = orc.compress_values(m)
    vt.ends[1] = 0  # non-monotone (ends[0] = 7 > 0)
    with pytest.raises(orc.IntegrityError):
        orc.validate(vt)
    with pytest.raises(orc.IntegrityError):
        orc.decompress(vt)
    pc = orc.compress_patterns(m)
    pc.row_pattern[3] = 99
    with pytest.raises(orc.IntegrityError):
        orc.validate(pc)
    with pytest.raises(orc.IntegrityError):
        orc.spmv(pc, np.ones(27))
    pc = orc.compress_patterns(m)
    pc.row_pattern[0] = 13  # interior pattern on a corner row -> column out of range
    with pytest.raises(orc.IntegrityError):
        orc.validate(pc)


# ---- K13/K14: byte model --
def test_k13_format_cost_and_roofline(orc):
    costs = [orc.format_cost(f, 27, 2).bytes_per_row for f in range(4)]
    assert costs == [324.0, 116.0, 12.0, 4.0]
    ell = orc.format_cost(orc.FMT_ELL, 27, 2)
    assert ell.bytes_per_flop == 6.0 and ell.flops_per_row == 54.0
    assert orc.required_bandwidth(11.6e9, ell) == pytest.approx(69.6e9)
    assert orc.required_bandwidth(12.5e9, ell) == pytest.approx(75e9)
    c6 = orc.format_cost(orc.FMT_ELL, 1, 1)
    assert orc.required_bandwidth(1.0, c6) == 6.0
    gf = [orc.roofline(orc.format_cost(f, 27, 2), 75e9)[0] / 1e9 for f in range(3)]
    assert gf[0] == pytest.approx(12.5) and gf[1] == pytest.approx(34.9, abs=0.05) and gf[2] == pytest.approx(337.5)
    assert abs(gf[1] - 34.8) / 34.8 < 0.01 and abs(gf[2] - 326) / 326 < 0.05  # acceptance 2
    assert orc.roofline(ell, 85e9)[0] / 1e9 == pytest.approx(14.17, abs=0.005)
    assert orc.roofline(ell, 150e9)[0] == 2 * orc.roofline(ell, 75e9)[0]
    f, lim = orc.roofline(ell, 75e9, peak_flops=1e9)
    assert (f, lim) == (1e9, "compute")
    assert orc.format_cost(orc.FMT_PATTERN_VALUES, 27, 2, include_input_vector=True).bytes_per_row == 12.0


def test_k14_measured_cost(orc):
    m = orc.generate_matrix(32, 32, 32)
    assert orc.measured_cost(orc.to_ell(m)).bytes_per_row == 324.0
    pv = orc.measured_cost(orc.compress_patterns(m, True)).bytes_per_row
    assert 4.0 < pv < 4.0 * 1.02
    p = orc.measured_cost(orc.compress_patterns(m, False)).bytes_per_row
    assert abs(p - 12.0) / 12.0 <= 0.02
    v = orc.measured_cost(orc.compress_values(m)).bytes_per_row
    assert v == 116.0
    one = orc.measured_cost(orc.compress_values(orc.generate_matrix(1, 1, 1)))
    assert one.bytes_per_row == 8.0
    assert orc.measured_cost(orc.to_ell(m)).flops_per_row == pytest.approx(2 * m.nnz / m.n)


# ---- the CG caller: SPEC.md:243-256,313-321, acceptance criterion 8 ----------
def test_dot_waxpby_examples(orc):
    assert orc.dot([1, 2], [3, 4]) == 11.0
    assert orc.dot(np.ones(1000), np.ones(1000)) == 1000.0
    x, y = np.array([1.0, 1.0]), np.array([1.0, 2.0])
    assert orc.waxpby(1, x, 0, y).tolist() == x.tolist() and orc.waxpby(0, x, 1, y).tolist() == y.tolist()
    assert orc.waxpby(2, x, 3, y).tolist() == [5.0, 8.0]
    with pytest.raises(orc.InvalidArgument):
        orc.dot([1, 2], [1, 2, 3])


def test_cg_examples(orc):
    m = orc.generate_matrix(1, 1, 1)
    x, it, conv, hist = orc.cg_solve(orc.to_ell(m), [52.0])
    assert x.tolist() == [2.0] and it == 1 and conv and hist[0] == 1.0
    m = orc.generate_matrix(16, 16, 16)
    b = orc.spmv(orc.to_ell(m), np.ones(m.n))
    results = [orc.cg_solve(f, b, tolerance=1e-8) for f in (orc.to_ell(m), orc.compress_values(m), orc.compress_patterns(m))]
    its = [r[1] for r in results]
    assert len(set(its)) == 1 and all(r[2] for r in results)  # identical iteration counts
    for x, it, conv, hist in results:
        assert np.abs(x - 1.0).max() <= 1e-6 and hist[-1] <= 1e-8 and len(hist) == it + 1
        assert np.abs(x - results[0][0]).max() <= 1e-9
        assert np.abs(hist - results[0][3]).max() <= 1e-10
    _, it, conv, _ = orc.cg_solve(orc.to_ell(m), b, max_iterations=1)
    assert it == 1 and not conv


# ---- symgs_sweep and the SymGS-preconditioned solve: SPEC.md:258-266, 308-311 ----------
def test_symgs_examples(orc):
    one = orc.generate_matrix(1, 1, 1)
    assert orc.symgs_sweep(one, [0.0], [52.0]).tolist() == [2.0]  # exact solve of the 1x1 system
    m = orc.generate_matrix(3, 3, 3)
    ell = orc.to_ell(m)
    b = orc.spmv(ell, np.ones(m.n))
    x = orc.symgs_sweep(m, np.zeros(m.n), b)
    assert np.linalg.norm(b - orc.spmv(ell, x)) < np.linalg.norm(b)  # the residual norm decreases
    assert np.array_equal(orc.symgs_sweep(m, np.zeros(m.n), b).view(np.uint64), x.view(np.uint64))  # deterministic
    # the definition, restated with a dense matrix: forward rows ascending, backward rows descending, latest values
    d, y = m.dense(), np.zeros(m.n)
    for order in (range(m.n), range(m.n - 1, -1, -1)):
        for i in order:
            s = 0.0
            for j in range(m.n):
                if j != i and d[i, j] != 0.0:
                    s = s + d[i, j] * y[j]
            y[i] = (b[i] - s) / d[i, i]
    assert np.array_equal(y.view(np.uint64), x.view(np.uint64))
    z = orc.csr_from_arrays(2, [0, 1, 2], [0, 1], [1.0, 0.0])  # zero diagonal: the singularity error
    with pytest.raises(orc.InvalidArgument):
        orc.symgs_sweep(z, [0.0, 0.0], [1.0, 1.0])
    with pytest.raises(orc.InvalidArgument):
        orc.symgs_sweep(m, np.zeros(3), b)


def test_symgs_preconditioned_cg(orc):
    m = orc.generate_matrix(12, 10, 8)
    ell = orc.to_ell(m)
    b = orc.spmv(ell, np.ones(m.n))
    x0, it0, conv0, _ = orc.cg_solve(ell, b)
    x1, it1, conv1, h1 = orc.cg_solve(ell, b, symgs_sweeps=1, matrix=m)
    assert conv0 and conv1 and it1 < it0  # the preconditioner pays
    assert np.abs(x1 - 1.0).max() <= 1e-6 and h1[0] == 1.0 and len(h1) == it1 + 1 and h1[-1] <= 1e-8
    for f in (orc.compress_values(m), orc.compress_patterns(m, True)):  # backend swap: same counts
        x2, it2, conv2, h2 = orc.cg_solve(f, b, symgs_sweeps=1, matrix=m)
        assert it2 == it1 and np.abs(x2 - x1).max() <= 1e-9 and np.abs(h2 - h1).max() <= 1e-10
    _, it3, _, _ = orc.cg_solve(ell, b, symgs_sweeps=2, matrix=m)
    assert it3 <= it1
