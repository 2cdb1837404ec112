"""z-slabs behind the C-ABI (spmvb_slab_* / spmvb_multi_*): G logical slabs on ONE device, the halo exchange as
same-device copies between the slabs' ghosted vectors -- the code path a multi-GPU box runs with peer copies -- must
reproduce the whole matrix bit for bit: ids (after the dictionary merge) and y.  Slabs run one after the other on their
own streams; none of them waits on another (x is quiescent during a SpMV)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    import paper_1612_00530_b200 as sp
    assert sp.device_count() >= 1
    return sp


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("g,G", [((64, 12, 10), 2), ((128, 10, 9), 3), ((256, 8, 16), 2), ((128, 20, 40), 4), ((72, 9, 7), 7),
                                 ((33, 5, 6), 2)])
def test_logical_slabs_equal_the_whole_matrix(sp, orc, g, G, mode):
    nx, ny, nz = g
    whole = orc.compress_patterns_grid(nx, ny, nz, values_in_pattern=True)
    x = orc.make_test_vector(whole.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
    ref = orc.spmv(whole, x)
    ms = sp.MultiSlab(sp.GridSpec(nx, ny, nz), [0] * G)
    assert ms.n_parts == G
    ms.fill_x(sp.RANDOM, 7, -1.0, 1.0)  # the seeded global vector, each slab its slice
    for rep in range(4):  # direct launches, graph capture, two replays
        ms.spmv(mode)
    ms.sync()
    y = ms.download_y()
    assert np.array_equal(bits(y), bits(ref))
    # per-slab streams equal the slice of a single-device compression (ids after the dictionary merge)
    plane = nx * ny
    for p in range(G):
        dev, z0, z1, a, xg, yg = ms.part(p)
        assert dev == 0 and a.info.row_offset == z0 * plane and a.info.n == (z1 - z0) * plane
        assert np.array_equal(a.download("row_pattern"), whole.row_pattern[z0 * plane:z1 * plane])
        assert a.download("disp_flat").tobytes() == whole.disp_flat.tobytes()
        assert a.download("ends_flat").tobytes() == whole.ends_flat.tobytes()


@pytest.mark.parametrize("fmt", ["ell", "vt"])
def test_logical_slabs_other_formats(sp, orc, fmt):
    nx, ny, nz, G = 40, 9, 11, 3
    m = orc.generate_matrix(nx, ny, nz)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=3, lo=-1.0, hi=1.0)
    ref = orc.spmv(orc.to_ell(m) if fmt == "ell" else orc.compress_values(m), x)
    ms = sp.MultiSlab(sp.GridSpec(nx, ny, nz), [0] * G, fmt=sp.FMT_ELL if fmt == "ell" else sp.FMT_VT)
    ms.upload_x(x)
    for mode in (0, 1, 0, 0):
        ms.spmv(mode)
    ms.sync()
    assert np.array_equal(bits(ms.download_y()), bits(ref))


def test_slabs_refuse_rows_that_reach_beyond_the_halo(sp, orc):
    """BASELINE config 4 adds entries at random in-bounds columns: such rows need more of x than the one-plane halo, so
    the perturbed grid cannot be cut into slabs (it is a single-GPU configuration).  A perturbation without added
    far columns can: noise only keeps every row inside the stencil's reach."""
    with pytest.raises(sp.InvalidArgument, match="beyond the one-plane halo"):
        sp.MultiSlab(sp.GridSpec(64, 16, 12), [0] * 3, perturb=(11, 0.1, 0.1), min_pattern_rows=2)


def test_slab_graph_replay_and_direct_launches_agree(sp, orc):
    nx, ny, nz = 128, 16, 24
    plane = nx * ny
    whole = orc.compress_patterns_grid(nx, ny, nz, values_in_pattern=True)
    x = orc.make_test_vector(whole.n, orc.RANDOM, seed=9, lo=-1.0, hi=1.0)
    ref = orc.spmv(whole, x)
    # the middle slab of three, driven through spmvb_slab_* directly; its neighbours' planes come from a full copy of x
    z0, z1 = 8, 16
    csr = sp.generate_matrix(sp.GridSpec(nx, ny, nz), row_begin=z0 * plane, row_end=z1 * plane)
    a = sp.compress_patterns(csr, True)
    # an interior slab numbers its 9 shapes by its own first occurrences: the same shapes row by row, other numbers (no merge here)
    def shapes_of(off, flat):
        return [tuple(flat[off[q]:off[q + 1]].tolist()) for q in range(len(off) - 1)]
    mine = shapes_of(a.download("disp_offsets"), a.download("disp_flat"))
    theirs = shapes_of(whole.disp_offsets, whole.disp_flat)
    to_whole = np.array([theirs.index(s) for s in mine], dtype=np.int32)
    assert np.array_equal(to_whole[a.download("row_pattern")], whole.row_pattern[z0 * plane:z1 * plane])
    slab = sp.Slab(a, plane, True, True)
    xfull = sp.DeviceVector.from_host(x)
    n = (z1 - z0) * plane
    xg = sp.DeviceVector.from_host(np.concatenate([np.full(plane, np.nan), x[z0 * plane:z1 * plane], np.full(plane, np.nan)]))
    lo_src = xfull.ptr + 8 * (z0 - 1) * plane
    hi_src = xfull.ptr + 8 * z1 * plane
    for graph in (1, 0):
        sp.set_option("slab_graph", graph)
        try:
            for mode in (sp.SLAB_SERIAL, sp.SLAB_OVERLAP):
                y = sp.DeviceVector.from_host(np.full(n, np.nan))
                used = []
                for _ in range(4):
                    slab.spmv(xg, y, lo_src, hi_src, mode)
                    used.append(slab.last_was_graph)
                assert used == ([False, True, True, True] if graph else [False] * 4)
                assert np.array_equal(bits(y.to_host()), bits(ref[z0 * plane:z1 * plane]))
        finally:
            sp.set_option("slab_graph", 1)
    # the halves for callers that exchange themselves (NCCL): ghosts already in place
    y = sp.DeviceVector.from_host(np.full(n, np.nan))
    slab.interior(xg, y)
    mid = y.to_host()
    assert np.all(np.isnan(mid[:plane])) and np.all(np.isnan(mid[-plane:]))
    slab.boundary(xg, y)
    assert np.array_equal(bits(y.to_host()), bits(ref[z0 * plane:z1 * plane]))
    with pytest.raises(sp.InvalidArgument):
        sp.Slab(a, plane + 1, True, True)


def test_multi_rejects_bad_arguments(sp):
    with pytest.raises(sp.InvalidArgument):
        sp.MultiSlab(sp.GridSpec(8, 8, 2), [0, 0, 0])  # more slabs than planes
    with pytest.raises(sp.InvalidArgument):
        sp.MultiSlab(sp.GridSpec(8, 8, 8), [0, 99])
    ms = sp.MultiSlab(sp.GridSpec(8, 8, 8), [0, 0])
    with pytest.raises(sp.InvalidArgument):
        ms.upload_x(np.zeros(5))
