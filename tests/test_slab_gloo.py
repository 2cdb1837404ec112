"""Multi-process (gloo, CPU) tests of the z-slab host logic: partitioning, ghost-plane
layout, halo exchange over torch.distributed, dictionary merge.  The local SpMV is the
CPU oracle here (the product has no CPU kernel); on GPUs the same SlabSpmv drives the
CUDA kernel with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1612_00530_b200.slab import SlabLayout, SlabSpmv, merge_dictionaries


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, grid, out_dir):
    from oracle import oracle as orc
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = grid
        L = SlabLayout(nx, ny, nz, rank, world)
        r0, r1 = L.row_range
        n_global = nx * ny * nz
        # per-slab compression (global columns, displacements against the global row id) ...
        csr = orc.generate_matrix(nx, ny, nz, row_begin=r0, row_end=r1)
        pc = orc.compress_patterns(csr, True, row_offset=r0)
        # ... then the dictionary merge every rank performs
        first = {}
        for i, pid in enumerate(pc.row_pattern.tolist()):
            first.setdefault(pid, i)
        mine = [(first[q] + r0,) + tuple(map(tuple, pc.pattern(q))) for q in range(pc.n_patterns)]
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        merged, maps = merge_dictionaries(gathered)
        ids = np.array(maps[rank], dtype=np.int32)[pc.row_pattern]
        # the merged result must equal the slice of the single-matrix compression
        whole = orc.compress_patterns_grid(nx, ny, nz, values_in_pattern=True)
        assert [tuple(map(tuple, whole.pattern(q))) for q in range(whole.n_patterns)] == [tuple(map(tuple, k)) for k in merged]
        assert np.array_equal(ids, whole.row_pattern[r0:r1])
        # local x: owned part from the global vector, ghosts poisoned until the exchange fills them
        xg = orc.make_test_vector(n_global, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
        x_local = torch.full((L.x_len,), float("nan"), dtype=torch.float64)
        L.owned(x_local).copy_(torch.from_numpy(xg[r0:r1]))
        if not L.has_lower:
            x_local[:L.plane] = 0.0  # never read: boundary rows have no entries below
        if not L.has_upper:
            x_local[L.plane + L.n_local:] = 0.0
        y_local = torch.full((L.n_local,), float("nan"), dtype=torch.float64)
        # slab handle = global dictionary + local ids: reuse the whole-matrix struct on the local range
        calls = []

        def kernel(xl, yl, b, e):
            calls.append((b, e))
            orc.spmv_rows(whole, xl.numpy(), _View(yl.numpy(), r0), r0 + b, r0 + e, x_col0=L.x_col0)

        SlabSpmv(L, kernel, dist).spmv(x_local, y_local)
        ref = orc.spmv(whole, xg)[r0:r1]
        assert np.array_equal(y_local.numpy().view(np.uint64), ref.view(np.uint64)), f"rank {rank}"
        # interior first (overlaps the exchange), then the boundary planes
        lo = min(L.plane, L.n_local) if L.has_lower else 0
        hi = max(L.n_local - L.plane, lo) if L.has_upper else L.n_local
        want = ([(lo, hi)] if hi > lo else []) + ([(0, lo)] if lo > 0 else []) + ([(hi, L.n_local)] if hi < L.n_local else [])
        assert calls == want, (calls, want)
        open(os.path.join(out_dir, f"ok{rank}"), "w").write("ok")
    finally:
        dist.destroy_process_group()


class _View:
    """Presents a local y array at global row indices to the oracle (which indexes y by row)."""

    def __init__(self, arr, r0):
        self.arr, self.r0 = arr, r0
        self.dtype, self.flags = arr.dtype, arr.flags

    @property
    def ctypes(self):
        import ctypes as C

        class P:
            def __init__(s, a):
                s.a = a

            def data_as(s, t):
                return C.c_void_p(s.a)
        return P(self.arr.ctypes.data - 8 * self.r0)


@pytest.mark.parametrize("world,grid", [(2, (6, 5, 8)), (2, (4, 4, 5)), (3, (5, 4, 7)), (2, (4, 3, 2))])
def test_slab_spmv_over_gloo(tmp_path, world, grid):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, grid, str(tmp_path)), nprocs=world, join=True)
    assert all((tmp_path / f"ok{r}").exists() for r in range(world))


def test_layout_partition():
    for nz, world in ((256, 8), (10, 3), (7, 7), (512, 4)):
        rows = []
        for r in range(world):
            L = SlabLayout(4, 3, nz, r, world)
            z0, z1 = L.z_range
            assert z1 > z0 and L.row_range == (z0 * 12, z1 * 12)
            assert L.x_col0 == z0 * 12 - 12 and L.x_len == L.n_local + 24
            rows.append(L.row_range)
        assert rows[0][0] == 0 and rows[-1][1] == 12 * nz
        assert all(a[1] == b[0] for a, b in zip(rows[:-1], rows[1:]))


def test_merge_dictionaries_orders_by_global_first_row():
    a = [(0, (0, 1), (1, 2)), (5, (-1, 0), (1, 2))]
    b = [(12, (-1, 0), (1, 2)), (10, (-1, 0, 1), (2, 3))]
    merged, maps = merge_dictionaries([a, b])
    assert merged == [((0, 1), (1, 2)), ((-1, 0), (1, 2)), ((-1, 0, 1), (2, 3))]
    assert maps == [[0, 1], [1, 2]]


def _cg_worker(rank, world, port, grid, out_dir):
    from oracle import oracle as orc
    from paper_1612_00530_b200.slab import SlabCg
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = grid
        L = SlabLayout(nx, ny, nz, rank, world)
        r0, r1 = L.row_range
        whole = orc.compress_patterns_grid(nx, ny, nz, values_in_pattern=True)
        xs = orc.make_test_vector(nx * ny * nz, orc.RANDOM, seed=3, lo=-1.0, hi=1.0)
        bg = orc.spmv(whole, xs)  # right-hand side with a known solution

        def kernel(xl, yl, b, e):
            orc.spmv_rows(whole, xl.numpy(), _View(yl.numpy(), r0), r0 + b, r0 + e, x_col0=L.x_col0)

        class Ops:  # the oracle's dot / waxpby on the owned rows
            @staticmethod
            def dot(u, v):
                return orc.dot(u.numpy(), v.numpy())

            @staticmethod
            def waxpby(alpha, x, beta, y, w):
                w.numpy()[:] = orc.waxpby(alpha, x.numpy(), beta, y.numpy())

        z = lambda n: torch.zeros(n, dtype=torch.float64)  # noqa: E731
        b_local = torch.from_numpy(bg[r0:r1].copy())
        x_local, r_local, ap_local, p_g = z(L.n_local), z(L.n_local), z(L.n_local), z(L.x_len)
        cg = SlabCg(L, SlabSpmv(L, kernel, dist), Ops, dist, torch)
        it, conv, hist = cg.solve(b_local, x_local, p_g, r_local, ap_local, max_iterations=200, tolerance=1e-10)
        x_ref, it_ref, conv_ref, hist_ref = orc.cg_solve(whole, bg, max_iterations=200, tolerance=1e-10)
        assert conv and conv_ref and it == it_ref, (it, it_ref)       # identical iteration counts
        assert np.allclose(hist, hist_ref, rtol=1e-6, atol=0.0)
        assert np.abs(x_local.numpy() - x_ref[r0:r1]).max() <= 1e-9 * np.abs(x_ref).max()
        assert np.abs(x_local.numpy() - xs[r0:r1]).max() <= 1e-7
        open(os.path.join(out_dir, f"cg{rank}"), "w").write("ok")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,grid", [(2, (6, 5, 8)), (3, (5, 4, 7))])
def test_slab_cg_over_gloo(tmp_path, world, grid):
    """Distributed CG: per-iteration halo exchange of the search direction + all_reduce of the three dots."""
    port = _free_port()
    mp.spawn(_cg_worker, args=(world, port, grid, str(tmp_path)), nprocs=world, join=True)
    assert all((tmp_path / f"cg{r}").exists() for r in range(world))
