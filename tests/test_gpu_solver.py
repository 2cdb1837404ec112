"""GPU tests of the CG caller: dot, waxpby and cg_solve on the device
against the oracle's restatement (acceptance criterion 8)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    import paper_1612_00530_b200 as sp
    return sp


def test_dot_and_waxpby(sp, orc):
    n = 1_000_003
    u = orc.make_test_vector(n, orc.RANDOM, seed=1, lo=-1.0, hi=1.0)
    v = orc.make_test_vector(n, orc.RANDOM, seed=2, lo=-1.0, hi=1.0)
    du, dv, dw = sp.DeviceVector.from_host(u), sp.DeviceVector.from_host(v), sp.DeviceVector(n)
    ref = orc.dot(u, v)
    got = sp.dot(du, dv)
    assert abs(got - ref) <= 1e-12 * np.abs(u * v).sum()  # tree vs index-ascending order
    assert sp.dot(du, dv) == got  # deterministic run to run
    assert sp.dot(sp.DeviceVector.from_host(np.ones(1000)), sp.DeviceVector.from_host(np.ones(1000))) == 1000.0
    sp.waxpby_into(0.75, du, -1.5, dv, dw)
    assert np.array_equal(dw.to_host().view(np.uint64), orc.waxpby(0.75, u, -1.5, v).view(np.uint64))  # bit-exact
    sp.waxpby_into(1.0, du, 2.0, dv, du)  # aliasing w = x
    assert np.array_equal(du.to_host().view(np.uint64), orc.waxpby(1.0, u, 2.0, v).view(np.uint64))


@pytest.mark.parametrize("g", [(16, 16, 16), (64, 20, 12)])
def test_cg_matches_the_oracle_on_every_backend(sp, orc, g):
    ref_m = orc.generate_matrix(*g)
    m = sp.generate_matrix(sp.GridSpec(*g))
    n = ref_m.n
    b = orc.spmv(orc.to_ell(ref_m), np.ones(n))
    db = sp.DeviceVector.from_host(b)
    x_ref, it_ref, conv_ref, hist_ref = orc.cg_solve(orc.to_ell(ref_m), b, tolerance=1e-8)
    assert conv_ref
    its, xs = [], []
    for a in (sp.to_ell(m), sp.compress_values(m), sp.compress_patterns(m, True)):
        x, rep = sp.cg_solve(a, db, tolerance=1e-8)
        xh = x.to_host()
        assert rep.converged and rep.final_residual() <= 1e-8
        assert rep.iterations == it_ref  # identical iteration counts
        assert len(rep.residual_history) == rep.iterations + 1 and rep.residual_history[0] == 1.0
        assert np.abs(np.array(rep.residual_history) - hist_ref).max() <= 1e-10
        assert np.abs(xh - 1.0).max() <= 1e-6 and np.abs(xh - x_ref).max() <= 1e-9
        assert rep.flops_total == rep.iterations * (2 * ref_m.nnz + 12 * n)
        its.append(rep.iterations)
        xs.append(xh)
    assert len(set(its)) == 1
    _, rep = sp.cg_solve(sp.to_ell(m), db, max_iterations=1)
    assert rep.iterations == 1 and not rep.converged


def test_cg_single_unknown_and_errors(sp, orc):
    a = sp.to_ell(sp.generate_matrix(sp.GridSpec(1, 1, 1)))
    x, rep = sp.cg_solve(a, sp.DeviceVector.from_host(np.array([52.0])))
    assert x.to_host().tolist() == [2.0] and rep.iterations == 1 and rep.converged
    with pytest.raises(sp.InvalidArgument):
        sp.cg_solve(a, sp.DeviceVector.from_host(np.array([52.0])), tolerance=0.0)
    # a singular system makes p.Ap = 0 -> non-finite alpha -> DivergenceError (solver.hpp:44)
    z = sp.upload_ell(2, 1, 0, np.zeros(2), np.array([0, 1], dtype=np.int32))
    with pytest.raises(sp._cabi.DivergenceError):
        sp.cg_solve(z, sp.DeviceVector.from_host(np.ones(2)))


@pytest.mark.parametrize("fmt", ["ell", "vt", "pattern", "hybrid"])
def test_cg_three_launch_iteration_keeps_the_bits(sp, orc, fmt):
    """"cg_fused_scalars": beta / stop flag / record by the last block of the vector kernel (1), alpha also formed at its head
    by every block and both kernels launched with programmatic stream serialization (2), against the separate alpha and beta
    kernels (0): the same reduction orders, so histories and solutions are bit-identical -- with and without the graph
    replay, converging and capped runs, repeated solves (the ticket counter returns to zero)."""
    g = (128, 12, 10) if fmt == "pattern" else (40, 9, 11)
    m = sp.generate_matrix(sp.GridSpec(*g))
    n = m.n
    a = {"ell": lambda: sp.to_ell(m), "vt": lambda: sp.compress_values(m), "pattern": lambda: sp.compress_patterns(m, True),
         "hybrid": lambda: sp.compress_patterns(sp.generate_matrix(sp.GridSpec(*g), perturb=(11, 0.1, 0.1)), True, min_pattern_rows=2)}[fmt]()
    b = sp.DeviceVector(n)
    sp.spmv_rows(sp.to_ell(m), sp.DeviceVector.from_host(np.ones(n)), b, 0, n)
    try:
        for graph in (1, 0):
            sp.set_option("cg_graph", graph)
            for cap, tol in ((300, 1e-10), (7, 1e-30), (1, 1e-30), (2, 1e-30)):
                got = []
                for fused in (1, 0, 2, 1):
                    sp.set_option("cg_fused_scalars", fused)
                    sp.set_option("cg_pdl", 1 if fused == 2 else 0)
                    x, rep = sp.cg_solve(a, b, max_iterations=cap, tolerance=tol)
                    got.append((x.to_host().view(np.uint64), rep))
                for xb, rep in got[1:]:
                    assert rep.iterations == got[0][1].iterations and rep.converged == got[0][1].converged
                    assert rep.residual_history == got[0][1].residual_history and np.array_equal(xb, got[0][0])
                if fmt != "hybrid" and cap == 300:
                    assert got[0][1].converged
    finally:
        sp.set_option("cg_graph", 1)
        sp.set_option("cg_fused_scalars", 1)
        sp.set_option("cg_pdl", 0)


@pytest.mark.parametrize("fmt", ["ell", "vt", "pattern", "hybrid"])
def test_cg_iteration_replayed_as_a_graph(sp, orc, fmt):
    """After the first iteration cg_solve replays its iteration as a CUDA graph ("cg_graph"): the same kernels in the same
    order, so the report and the solution are bit-identical to direct launches, on every backend."""
    g = (72, 10, 9)
    m = sp.generate_matrix(sp.GridSpec(*g), perturb=(11, 0.1, 0.1) if fmt == "hybrid" else None)
    n = m.n
    ell = sp.to_ell(m)
    a = {"ell": lambda: ell, "vt": lambda: sp.compress_values(sp.generate_matrix(sp.GridSpec(*g))),
         "pattern": lambda: sp.compress_patterns(m, True),
         "hybrid": lambda: sp.compress_patterns(m, True, min_pattern_rows=2)}[fmt]()
    b = sp.DeviceVector(n)
    sp.spmv_rows(ell if fmt != "vt" else a, sp.DeviceVector.from_host(np.ones(n)), b, 0, n)
    out = {}
    try:
        for graph in (0, 1, 1):
            sp.set_option("cg_graph", graph)
            x, rep = sp.cg_solve(a, b, max_iterations=40, tolerance=1e-9)  # (the perturbed matrix is not SPD: no convergence asked)
            assert sp.get_option("last_cg_graph") == graph and rep.iterations > 8
            out.setdefault(graph, []).append((x.to_host().view(np.uint64), rep))
        for cap in (1, 2, 3, 7):  # around the point where the graph takes over
            reps = []
            for graph in (0, 1):
                sp.set_option("cg_graph", graph)
                x, rep = sp.cg_solve(a, b, max_iterations=cap, tolerance=1e-9)
                reps.append((x.to_host().view(np.uint64), rep))
            assert reps[0][1].residual_history == reps[1][1].residual_history and np.array_equal(reps[0][0], reps[1][0])
            assert reps[1][1].iterations == cap
    finally:
        sp.set_option("cg_graph", 1)
    (x0, r0), (x1, r1), (x2, r2) = out[0][0], out[1][0], out[1][1]
    assert r0.iterations == r1.iterations == r2.iterations and r0.residual_history == r1.residual_history == r2.residual_history
    assert np.array_equal(x0, x1) and np.array_equal(x1, x2)


def test_cg_workspace_on_the_handle_and_run_ahead(sp, orc):
    """Repeated solves reuse the work vectors kept on the handle ("cg_keep_workspace"); with or without them, and wherever
    the stop falls relative to the host's run-ahead of four iterations, the report and the solution are identical."""
    g = (20, 12, 10)
    m = sp.generate_matrix(sp.GridSpec(*g))
    n = m.n
    a = sp.compress_patterns(m, True)
    ell = sp.to_ell(m)
    b = sp.DeviceVector(n)
    sp.spmv_rows(ell, sp.DeviceVector.from_host(np.ones(n)), b, 0, n)
    x0, rep0 = sp.cg_solve(a, b, tolerance=1e-9)
    assert rep0.converged and rep0.iterations > 6
    base = x0.to_host().view(np.uint64)
    try:
        for keep in (1, 0, 1):
            sp.set_option("cg_keep_workspace", keep)
            for _ in range(2):
                x, rep = sp.cg_solve(a, b, tolerance=1e-9)
                assert rep.iterations == rep0.iterations and rep.residual_history == rep0.residual_history
                assert np.array_equal(x.to_host().view(np.uint64), base)
    finally:
        sp.set_option("cg_keep_workspace", 1)
    # max_iterations below, at and above the run-ahead depth, and one past convergence: same prefix of the history
    for cap in (1, 2, 3, 4, 5, 6, rep0.iterations - 1, rep0.iterations, rep0.iterations + 1, rep0.iterations + 7):
        x, rep = sp.cg_solve(a, b, max_iterations=cap, tolerance=1e-9)
        k = min(cap, rep0.iterations)
        assert rep.iterations == k and rep.converged == (cap >= rep0.iterations)
        assert rep.residual_history == rep0.residual_history[: k + 1]
        if cap >= rep0.iterations:
            assert np.array_equal(x.to_host().view(np.uint64), base)  # nothing queued past the stop touched x
    # an interleaved solve on another handle does not disturb this one's vectors
    xe, repe = sp.cg_solve(ell, b, tolerance=1e-9)
    x, rep = sp.cg_solve(a, b, tolerance=1e-9)
    assert np.array_equal(x.to_host().view(np.uint64), base) and repe.iterations == rep0.iterations


@pytest.mark.parametrize("g", [(192, 6, 9), (128, 10, 8), (256, 6, 14), (72, 6, 9)])
def test_cg_takes_p_ap_from_the_tensor_ring_kernel(sp, orc, g):
    """Pattern format, whole square grid, tensor ring: p.Ap comes out of the SpMV kernel (one partial per warp, rows in
    schedule order).  Against the stand-alone dot: same iteration count, histories within 1e-12, solutions within 1e-12;
    deterministic run to run.  Grids whose lines end in a left-over column (128, 192, 256: per-warp, per-warp and per-CTA schedules) and one that does not (72)."""
    m = sp.generate_matrix(sp.GridSpec(*g))
    n = m.n
    a = sp.compress_patterns(m, True)
    b = sp.DeviceVector(n)
    sp.spmv_rows(sp.to_ell(m), sp.DeviceVector.from_host(np.ones(n)), b, 0, n)
    try:
        sp.set_option("cg_fused_dot", 0)
        x0, rep0 = sp.cg_solve(a, b, tolerance=1e-9)
        assert sp.get_option("last_cg_fused_dot") == 0
        sp.set_option("cg_fused_dot", 1)
        x1, rep1 = sp.cg_solve(a, b, tolerance=1e-9)
        assert sp.get_option("last_cg_fused_dot") == 1 and sp.get_option("last_pattern_kernel") == 9
        x2, rep2 = sp.cg_solve(a, b, tolerance=1e-9)
    finally:
        sp.set_option("cg_fused_dot", 1)
    assert rep0.converged and rep1.converged and rep1.iterations == rep0.iterations
    assert np.abs(np.array(rep1.residual_history) - np.array(rep0.residual_history)).max() <= 1e-12
    assert np.abs(x1.to_host() - x0.to_host()).max() <= 1e-12 and np.abs(x1.to_host() - 1.0).max() <= 1e-6
    assert rep2.residual_history == rep1.residual_history and np.array_equal(x2.to_host().view(np.uint64), x1.to_host().view(np.uint64))
    # hybrid handles (exception rows go through another kernel) and the other formats keep the stand-alone dot
    xe, repe = sp.cg_solve(sp.to_ell(m), b, tolerance=1e-9)
    assert sp.get_option("last_cg_fused_dot") == 0 and repe.iterations == rep0.iterations


@pytest.mark.parametrize("g", [(1, 1, 1), (3, 3, 3), (5, 4, 3), (16, 7, 2), (1, 6, 4), (4, 1, 1), (33, 9, 5), (20, 20, 20)])
def test_symgs_sweep_by_hyperplanes_is_the_sequential_sweep(sp, orc, g):
    """symgs_sweep (kernels.hpp:44-48) on the device: rows by hyperplanes ix + 2 iy + 4 iz, bit-identical to the oracle's
    sequential natural-order sweep, for a random start and right-hand side, twice in a row."""
    m = orc.generate_matrix(*g)
    n = m.n
    dm = sp.generate_matrix(sp.GridSpec(*g))
    x = orc.make_test_vector(n, orc.RANDOM, seed=3, lo=-1.0, hi=1.0)
    b = orc.make_test_vector(n, orc.RANDOM, seed=4, lo=-1.0, hi=1.0)
    dx, db = sp.DeviceVector.from_host(x), sp.DeviceVector.from_host(b)
    for _ in range(2):
        x = orc.symgs_sweep(m, x, b)
        sp.symgs_sweep(dm, sp.GridSpec(*g), dx, db)
        assert np.array_equal(dx.to_host().view(np.uint64), x.view(np.uint64))


@pytest.mark.parametrize("g,served", [((3, 3, 3), True), ((5, 4, 3), True), ((33, 9, 5), True), ((20, 20, 20), True), ((64, 3, 2), True),
                                      ((8, 8, 300), True),     # more planes than SMs: a CTA takes several planes, round-robin
                                      ((9, 200, 150), True),   # ... with lines on seven of the eight warps
                                      ((40, 257, 3), False),   # lines longer than a CTA: the grid-barrier kernel
                                      ((2, 5, 4), False), ((7, 2, 6), False)])  # too narrow for the box decode
def test_symgs_plane_pipeline_and_its_fallbacks(sp, orc, g, served):
    """The plane-per-CTA pipeline (box masks, operands through shared-memory rings, release / acquire clocks between planes) and the
    kernels it falls back to are the oracle's sequential sweep bit for bit, whatever the lag between planes."""
    m = orc.generate_matrix(*g)
    dm = sp.generate_matrix(sp.GridSpec(*g))
    x0 = orc.make_test_vector(m.n, orc.RANDOM, seed=13, lo=-1.0, hi=1.0)
    b = orc.make_test_vector(m.n, orc.RANDOM, seed=14, lo=-1.0, hi=1.0)
    ref = orc.symgs_sweep(m, orc.symgs_sweep(m, x0, b), b)
    db = sp.DeviceVector.from_host(b)
    for pipeline, lag in ((1, 0), (1, 9), (0, 0)):
        sp.set_option("symgs_pipeline", pipeline)
        sp.set_option("symgs_lag", lag)
        try:
            dx = sp.DeviceVector.from_host(x0)
            for _ in range(2):
                sp.symgs_sweep(dm, sp.GridSpec(*g), dx, db)
            assert sp.get_option("last_symgs_kernel") == (2 if pipeline and served else 1)
        finally:
            sp.set_option("symgs_pipeline", 1)
            sp.set_option("symgs_lag", 0)
        assert np.array_equal(dx.to_host().view(np.uint64), ref.view(np.uint64)), (pipeline, lag)


def test_symgs_sweeps_on_two_streams_from_two_host_threads(sp, orc):
    """Sweeps of different handles enqueued from two host threads on two streams of one device: each has its own synchronisation
    words (per device and stream), so in whatever order the device runs them every one is the oracle's sweep bit for bit."""
    import threading
    import torch
    errors = []
    cases = []
    for g in ((20, 20, 20), (33, 9, 5)):
        m = orc.generate_matrix(*g)
        x0 = orc.make_test_vector(m.n, orc.RANDOM, seed=21, lo=-1.0, hi=1.0)
        b = orc.make_test_vector(m.n, orc.RANDOM, seed=22, lo=-1.0, hi=1.0)
        ref = x0
        for _ in range(6):
            ref = orc.symgs_sweep(m, ref, b)
        cases.append((g, sp.generate_matrix(sp.GridSpec(*g)), x0, sp.DeviceVector.from_host(b), ref, torch.cuda.Stream()))

    def sweeps(g, dm, dx, db, st, pipeline):
        try:
            sp.check(sp.lib.spmvb_set_device(0))  # options and the current device are per host thread
            sp.set_option("symgs_pipeline", pipeline)
            for _ in range(6):
                sp.symgs_sweep(dm, sp.GridSpec(*g), dx, db, stream=st)
            st.synchronize()
        except Exception as ex:  # noqa: BLE001
            errors.append(ex)

    for pipeline in (1, 0):
        xs = [sp.DeviceVector.from_host(c[2]) for c in cases]  # every round starts from the same x
        threads = [threading.Thread(target=sweeps, args=(c[0], c[1], dx, c[3], c[5], pipeline)) for c, dx in zip(cases, xs)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        assert not errors, errors
        for c, dx in zip(cases, xs):
            assert np.array_equal(dx.to_host().view(np.uint64), c[4].view(np.uint64)), (c[0], pipeline)


def test_symgs_examples_and_refusals(sp, orc):
    one = sp.generate_matrix(sp.GridSpec(1, 1, 1))
    dx = sp.DeviceVector.from_host(np.array([0.0]))
    sp.symgs_sweep(one, sp.GridSpec(1, 1, 1), dx, sp.DeviceVector.from_host(np.array([52.0])))
    assert dx.to_host().tolist() == [2.0]
    # user-supplied values, explicit rows of a sparser stencil (7-point): still ordered by the hyperplanes
    g = (6, 5, 4)
    gs = sp.GridSpec(*g)
    rows = []
    for iz in range(g[2]):
        for iy in range(g[1]):
            for ix in range(g[0]):
                r = [(gs.node(ix, iy, iz), 6.5)]
                for dx_, dy_, dz_ in ((-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)):
                    jx, jy, jz = ix + dx_, iy + dy_, iz + dz_
                    if 0 <= jx < g[0] and 0 <= jy < g[1] and 0 <= jz < g[2]:
                        r.append((gs.node(jx, jy, jz), -1.0 - 0.01 * (jx + jy)))
                rows.append(sorted(r))
    m7 = orc.stencil_from_rows(gs.rows(), rows)
    d7 = sp.stencil_from_rows(gs.rows(), rows)
    x = np.linspace(-1.0, 1.0, gs.rows())
    b = np.cos(np.arange(gs.rows()))
    dx, db = sp.DeviceVector.from_host(x), sp.DeviceVector.from_host(b)
    sp.symgs_sweep(d7, gs, dx, db)
    assert sp.get_option("last_symgs_kernel") == 2  # a sub-box of the 27 neighbours per row: the plane pipeline
    assert np.array_equal(dx.to_host().view(np.uint64), orc.symgs_sweep(m7, x, b).view(np.uint64))
    # refusals leave x untouched: zero diagonal (singularity); a coupling the schedule does not order; wrong grid
    before = dx.to_host().copy()
    z = sp.upload_csr(2, [0, 1, 2], [0, 1], [1.0, 0.0])
    two = sp.DeviceVector.from_host(np.zeros(2))
    with pytest.raises(sp.InvalidArgument, match="diagonal"):
        sp.symgs_sweep(z, sp.GridSpec(2, 1, 1), two, two)
    # couplings outside the 27-point box are swept exactly as long as the hyperplanes order them the way the row index does
    far = [list(r) for r in rows]
    far[0] = sorted(far[0] + [(gs.rows() - 1, -0.5)])
    far[-1] = sorted(far[-1] + [(0, -0.5)])
    far[3] = sorted(far[3] + [(3 + 2 * g[0] - 1, -0.25)])  # node (3,0,0) -> (2,2,0): higher index, higher level
    dfar, xf = sp.DeviceVector.from_host(x), orc.symgs_sweep(orc.stencil_from_rows(gs.rows(), far), x, b)
    sp.symgs_sweep(sp.stencil_from_rows(gs.rows(), far), gs, dfar, db)
    assert sp.get_option("last_symgs_kernel") == 1  # rows that are no sub-boxes: the general kernel
    assert np.array_equal(dfar.to_host().view(np.uint64), xf.view(np.uint64))
    bad = [list(r) for r in rows]
    bad[5] = sorted(bad[5] + [(6, -0.25)])  # node (5,0,0), level 5 -> node (0,1,0): higher index but level 2
    with pytest.raises(sp.InvalidArgument, match="hyperplane"):
        sp.symgs_sweep(sp.stencil_from_rows(gs.rows(), bad), gs, dx, db)
    with pytest.raises(sp.InvalidArgument):
        sp.symgs_sweep(d7, sp.GridSpec(6, 5, 5), dx, db)
    with pytest.raises(sp.InvalidArgument):
        sp.symgs_sweep(sp.to_ell(d7), gs, dx, db)  # the sweep runs on the uncompressed matrix only (SPEC.md DESIGN DECISIONS)
    assert np.array_equal(dx.to_host().view(np.uint64), before.view(np.uint64))


@pytest.mark.parametrize("g", [(12, 10, 8), (16, 16, 16)])
def test_symgs_preconditioned_cg_matches_the_oracle(sp, orc, g):
    """cg_solve with the SymGS preconditioner (solver.hpp:40-46): iteration counts identical to the oracle's on
    every backend, histories within 1e-10, solutions within 1e-9; fewer iterations than without it; analytic flop count."""
    ref_m = orc.generate_matrix(*g)
    gs = sp.GridSpec(*g)
    m = sp.generate_matrix(gs)
    n = ref_m.n
    b = orc.spmv(orc.to_ell(ref_m), np.ones(n))
    db = sp.DeviceVector.from_host(b)
    for sweeps in (1, 2):
        x_ref, it_ref, conv_ref, hist_ref = orc.cg_solve(orc.to_ell(ref_m), b, symgs_sweeps=sweeps, matrix=ref_m)
        assert conv_ref
        for a in (sp.to_ell(m), sp.compress_values(m), sp.compress_patterns(m, True)):
            x, rep = sp.cg_solve(a, db, symgs_sweeps=sweeps, csr=m, grid=gs)
            assert rep.converged and rep.iterations == it_ref
            assert np.abs(np.array(rep.residual_history) - hist_ref).max() <= 1e-10
            assert np.abs(x.to_host() - x_ref).max() <= 1e-9 and np.abs(x.to_host() - 1.0).max() <= 1e-6
            assert rep.flops_total == it_ref * (2 * ref_m.nnz + 12 * n) + it_ref * sweeps * 4 * ref_m.nnz  # SPEC.md:321 + symgs_flops
    _, plain = sp.cg_solve(sp.to_ell(m), db)
    _, pre = sp.cg_solve(sp.to_ell(m), db, symgs_sweeps=1, csr=m, grid=gs)
    assert pre.iterations < plain.iterations
    _, one = sp.cg_solve(sp.to_ell(m), db, symgs_sweeps=1, csr=m, grid=gs, max_iterations=1)
    assert one.iterations == 1 and not one.converged
    with pytest.raises(sp.InvalidArgument):
        sp.cg_solve(sp.to_ell(m), db, symgs_sweeps=1)


def test_slab_cg_driver_on_the_device(sp, orc):
    """The distributed CG driver (slab.py:SlabCg) with the CUDA kernels as its operations, one slab: the same iteration
    count and history as the single-call device solver, and the known solution."""
    import torch
    g = (128, 12, 10)
    L = sp.SlabLayout(*g, 0, 1)
    n = L.n_local
    pc = sp.build_slab_pattern(sp, L, None, keep_csr=False)
    xs = orc.make_test_vector(n, orc.RANDOM, seed=3, lo=-1.0, hi=1.0)
    ref = orc.compress_patterns_grid(*g, values_in_pattern=True)
    b = orc.spmv(ref, xs)

    class Ops:
        @staticmethod
        def dot(u, v):
            out = sp.C.c_double()
            sp.check(sp.lib.spmvb_dot(sp.C.c_void_p(u.data_ptr()), sp.C.c_void_p(v.data_ptr()), u.numel(), sp.C.byref(out), None))
            return out.value

        @staticmethod
        def waxpby(alpha, x, beta, y, w):
            sp.check(sp.lib.spmvb_waxpby(alpha, sp.C.c_void_p(x.data_ptr()), beta, sp.C.c_void_p(y.data_ptr()),
                                         sp.C.c_void_p(w.data_ptr()), x.numel(), None))

    def kernel(xl, yl, b0, e0):
        sp.spmv_rows(pc, xl, yl, b0, e0, x_col0=L.x_col0, x_len=L.x_len)

    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    z = lambda k: torch.zeros(k, dtype=torch.float64, device="cuda")  # noqa: E731
    b_d, x_d, r_d, ap_d, p_g = dev(b), z(n), z(n), z(n), z(L.x_len)
    cg = sp.SlabCg(L, sp.SlabSpmv(L, kernel), Ops, None, torch)
    it, conv, hist = cg.solve(b_d, x_d, p_g, r_d, ap_d, max_iterations=300, tolerance=1e-10)
    torch.cuda.synchronize()
    x1, rep = sp.cg_solve(sp.upload_pattern(ref.n, ref.table, ref.disp_offsets, ref.disp_flat, ref.ends_flat, ref.row_pattern, True),
                          sp.DeviceVector.from_host(b), max_iterations=300, tolerance=1e-10)
    assert conv and rep.converged and it == rep.iterations
    assert np.allclose(hist, rep.residual_history, rtol=1e-9, atol=0.0)
    assert np.abs(x_d.cpu().numpy() - xs).max() <= 1e-7
