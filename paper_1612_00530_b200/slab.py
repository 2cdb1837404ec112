"""z-slab multi-GPU SpMV: one process per GPU, one-plane halo of x exchanged with
the z-neighbours each SpMV (torch.distributed send/recv: NCCL over NVLink on
GPUs, gloo in the CPU tests), overlapped with the rows that need no halo.

Partitioning: with x-fastest numbering a z-slab is a
contiguous row range [z0*plane, z1*plane) -- exactly the [begin,end) that
unchecked::spmv_rows (kernels.hpp:27-36) already takes.  Rank r keeps
x_local = [ghost plane below | owned planes | ghost plane above]; a global column
c lives at x_local[c - x_col0] with x_col0 = (z0-1)*plane.  Displacements are
translation invariant, so the global dictionary and the slice of the global
row_pattern are used unchanged: per-slab streams are bit-identical to the slice
of a single-device compression (ids after the dictionary merge below).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class SlabLayout:
    """Rows and ghost planes of one rank."""
    nx: int
    ny: int
    nz_global: int
    rank: int
    world: int

    @property
    def plane(self):
        return self.nx * self.ny

    @property
    def z_range(self):
        """Planes [z0,z1): nz_global split as evenly as possible, low ranks get the remainder."""
        base, rem = divmod(self.nz_global, self.world)
        z0 = self.rank * base + min(self.rank, rem)
        return z0, z0 + base + (1 if self.rank < rem else 0)

    @property
    def row_range(self):
        z0, z1 = self.z_range
        return z0 * self.plane, z1 * self.plane

    @property
    def n_local(self):
        r0, r1 = self.row_range
        return r1 - r0

    @property
    def has_lower(self):
        return self.rank > 0

    @property
    def has_upper(self):
        return self.rank < self.world - 1

    @property
    def x_col0(self):
        """Global column of x_local[0]; the ghost slot below is allocated even on rank 0."""
        return self.row_range[0] - self.plane

    @property
    def x_len(self):
        return self.n_local + 2 * self.plane

    def owned(self, x_local):
        return x_local[self.plane:self.plane + self.n_local]


def merge_dictionaries(local_dicts):
    """Merge per-slab dictionaries into the numbering a single-matrix compression issues:
    ids by first occurrence in ascending GLOBAL row order.

    local_dicts: per rank, a list of (first_global_row, displacements tuple, ends tuple).
    Returns (merged list of (displacements, ends), per-rank old->new id maps)."""
    best = {}
    for d in local_dicts:
        for first, disp, ends in d:
            key = (tuple(disp), tuple(ends))
            if key not in best or first < best[key]:
                best[key] = first
    order = sorted(best, key=lambda k: best[k])
    new_id = {k: i for i, k in enumerate(order)}
    maps = [[new_id[(tuple(disp), tuple(ends))] for _, disp, ends in d] for d in local_dicts]
    return order, maps


class SlabSpmv:
    """y_local = (A x)[slab rows] with the halo exchange overlapped with interior rows.

    kernel(x_local, y_local, begin, end) computes local rows [begin,end); the product
    passes the CUDA spmv_rows, the CPU tests inject the oracle's.  `dist` is
    torch.distributed (or None for a single slab)."""

    def __init__(self, layout: SlabLayout, kernel, dist=None, comm_stream=None, main_stream=None, torch=None,
                 two_stream_boundaries=False):
        """two_stream_boundaries: kernel accepts a `stream=` keyword; the lower boundary plane then runs on the side stream."""
        self.L, self.kernel, self.dist = layout, kernel, dist
        self.comm_stream, self.main_stream, self.torch = comm_stream, main_stream, torch
        self.two_stream_boundaries = two_stream_boundaries and comm_stream is not None

    def _exchange_ops(self, x_local):
        L, d = self.L, self.dist
        p, n = L.plane, L.n_local
        ops = []
        if L.has_lower:  # my first owned plane -> lower neighbour's upper ghost; its last plane -> my lower ghost
            ops.append(d.P2POp(d.isend, x_local[p:2 * p], L.rank - 1))
            ops.append(d.P2POp(d.irecv, x_local[0:p], L.rank - 1))
        if L.has_upper:
            ops.append(d.P2POp(d.isend, x_local[n:n + p], L.rank + 1))
            ops.append(d.P2POp(d.irecv, x_local[n + p:n + 2 * p], L.rank + 1))
        return ops

    def exchange(self, x_local):
        """Blocking halo exchange (used by tests and as the non-overlapped baseline)."""
        if self.dist is None or self.L.world == 1:
            return
        for r in self.dist.batch_isend_irecv(self._exchange_ops(x_local)):
            r.wait()

    def spmv(self, x_local, y_local):
        """One SpMV: exchange || interior rows, then the first and last owned planes."""
        L = self.L
        p, n = L.plane, L.n_local
        if self.dist is None or L.world == 1:
            self.kernel(x_local, y_local, 0, n)
            return
        lo = min(p, n) if L.has_lower else 0        # rows [0,lo) need the lower ghost
        hi = max(n - p, lo) if L.has_upper else n   # rows [hi,n) need the upper ghost
        if self.comm_stream is not None:
            t = self.torch
            self.comm_stream.wait_stream(self.main_stream)  # x_local is ready
            with t.cuda.stream(self.comm_stream):
                reqs = self.dist.batch_isend_irecv(self._exchange_ops(x_local))
            if hi > lo:
                self.kernel(x_local, y_local, lo, hi)       # interior rows overlap the exchange
            with t.cuda.stream(self.comm_stream):
                for r in reqs:
                    r.wait()
            if self.two_stream_boundaries and lo > 0 and hi < n:
                # the two boundary planes are independent: one goes on the side stream right behind the receive, the
                # other on the main stream, so that they share the GPU once the interior kernel has drained
                self.kernel(x_local, y_local, 0, lo, stream=self.comm_stream)
                self.main_stream.wait_stream(self.comm_stream)  # (the receive; the lower plane is ordered by the final wait)
                self.kernel(x_local, y_local, hi, n)
                self.main_stream.wait_stream(self.comm_stream)
                return
            self.main_stream.wait_stream(self.comm_stream)
        else:
            reqs = self.dist.batch_isend_irecv(self._exchange_ops(x_local))
            if hi > lo:
                self.kernel(x_local, y_local, lo, hi)
            for r in reqs:
                r.wait()
        if lo > 0:
            self.kernel(x_local, y_local, 0, lo)
        if hi < n:
            self.kernel(x_local, y_local, hi, n)


class DeviceSlabSpmv(SlabSpmv):
    """The product's z-slab SpMV of one rank: the kernels and, where the neighbours' memory is mapped, the exchange run
    behind the C-ABI (spmvb_slab_*, csrc/slab.cu); torch.distributed carries the exchange otherwise.

    exchange = "nccl": the two boundary planes travel by batch_isend_irecv (NCCL send/recv over NVLink).
               schedule "serial": exchange, then ONE launch over all owned planes; "overlap": exchange on the side stream
               while the planes that need no ghost are computed, then the first and last owned plane.
    exchange = "p2p":  every rank maps its neighbours' vectors (CUDA IPC) and spmvb_slab_spmv pulls their boundary planes
               with two copies in front of the launch, all of it one CUDA graph per SpMV.  x must be quiescent on the
               neighbours during the call (true for a fixed x; CG orders it with its all-reduces plus `fence()`).
    `x_local` must come from spmvb_vec_alloc (DeviceVector) for "p2p"."""

    def __init__(self, sp, layout: SlabLayout, matrix, dist, main_stream, comm_stream, torch, exchange="nccl", schedule="serial"):
        super().__init__(layout, None, dist, comm_stream, main_stream, torch)
        if exchange not in ("nccl", "p2p") or schedule not in ("serial", "overlap"):
            raise ValueError(f"unknown exchange / schedule: {exchange} / {schedule}")
        self.sp, self.exchange_kind, self.schedule = sp, exchange, schedule
        self.slab = sp.Slab(matrix, layout.plane, layout.has_lower, layout.has_upper)
        self.mode = sp.SLAB_SERIAL if schedule == "serial" else sp.SLAB_OVERLAP
        self._peers = {}      # rank -> mapped base pointer of its x_local
        self._graph = None    # a captured step of the "nccl" exchange (torch.cuda.CUDAGraph), when capture worked
        self._graph_key = None
        self.launches_per_spmv = 1 if (schedule == "serial" or layout.world == 1) else 1 + int(layout.has_lower) + int(layout.has_upper)

    # -- "p2p": map the neighbours' x_local once
    def map_neighbours(self, x_local):
        L, d, sp = self.L, self.dist, self.sp
        handles = [None] * L.world
        d.all_gather_object(handles, sp.ipc_export(x_local))
        for r in (L.rank - 1, L.rank + 1):
            if 0 <= r < L.world:
                self._peers[r] = sp.ipc_open(handles[r])
        self._mapped_for = x_local.data_ptr()

    def fence(self):
        """"p2p" only: every rank's producers of x_local have completed before anyone pulls a plane of it -- a stream
        synchronize and a barrier.  A caller whose x changes between SpMVs (CG's search direction) calls it before each
        spmv(); the all-reduce that follows the SpMV orders the pulls before the next update of x."""
        if self.exchange_kind == "p2p" and self.dist is not None and self.L.world > 1:
            self.main_stream.synchronize()
            self.dist.barrier()

    def unmap_neighbours(self):
        for ptr in self._peers.values():
            self.sp.ipc_close(ptr)
        self._peers = {}

    def _sources(self):
        L = self.L
        z = [SlabLayout(L.nx, L.ny, L.nz_global, r, L.world) for r in (L.rank - 1, L.rank + 1)]
        lo = self._peers[L.rank - 1] + 8 * z[0].n_local if L.has_lower else None     # its last owned plane (skip its lower ghost)
        hi = self._peers[L.rank + 1] + 8 * L.plane if L.has_upper else None           # its first owned plane
        return lo, hi

    def _step_nccl(self, x_local, y_local):
        L, t = self.L, self.torch
        if self.schedule == "serial":
            for r in self.dist.batch_isend_irecv(self._exchange_ops(x_local)):
                r.wait()
            self.slab.spmv(x_local, y_local, None, None, self.mode, stream=t.cuda.current_stream())
            return
        cur = t.cuda.current_stream()
        self.comm_stream.wait_stream(cur)
        with t.cuda.stream(self.comm_stream):
            reqs = self.dist.batch_isend_irecv(self._exchange_ops(x_local))
        self.slab.interior(x_local, y_local, stream=cur)
        with t.cuda.stream(self.comm_stream):
            for r in reqs:
                r.wait()
        cur.wait_stream(self.comm_stream)
        self.slab.boundary(x_local, y_local, stream=cur)

    def capture(self, x_local, y_local):
        """Record one step of the "nccl" exchange + launches into a CUDA graph (NCCL operations are capturable); call
        after at least one eager step (communicators and kernel attributes exist).  False when capture is not possible."""
        t = self.torch
        if self.exchange_kind != "nccl" or self.L.world == 1:
            return False
        try:
            g = t.cuda.CUDAGraph()
            with t.cuda.graph(g, stream=self.main_stream, capture_error_mode="thread_local"):
                self._step_nccl(x_local, y_local)
            self._graph, self._graph_key = g, (x_local.data_ptr(), y_local.data_ptr())
            return True
        except Exception:  # noqa: BLE001 -- any failure leaves the eager path
            self._graph = None
            return False

    def spmv(self, x_local, y_local):
        L, t = self.L, self.torch
        if self.dist is None or L.world == 1:
            self.slab.spmv(x_local, y_local, None, None, self.sp.SLAB_SERIAL, stream=self.main_stream)
            return
        if self.exchange_kind == "p2p":
            if not self._peers or self._mapped_for != x_local.data_ptr():
                self.map_neighbours(x_local)
            lo, hi = self._sources()
            self.slab.spmv(x_local, y_local, lo, hi, self.mode, stream=self.main_stream)
            return
        if self._graph is not None and self._graph_key == (x_local.data_ptr(), y_local.data_ptr()):
            with t.cuda.stream(self.main_stream):
                self._graph.replay()
            return
        with t.cuda.stream(self.main_stream):
            self._step_nccl(x_local, y_local)


class SlabCg:
    """Unpreconditioned CG (solver.hpp:40-46) over z-slabs: the SpMV is SlabSpmv (halo of the search
    direction exchanged every iteration, overlapped with the interior rows), the three dots of an iteration are local
    dots summed over the ranks with one all_reduce each, the three waxpbys are local.  x0 = 0; stops when
    ||r||2 / ||b||2 <= tolerance.  Same operation sequence as the single-device `cg_solve`, so iteration counts agree
    across backends; the dot products are summed in a different order, so the iterates agree to rounding.

    ops.dot(u, v) -> float and ops.waxpby(alpha, x, beta, y, w) work on owned-row vectors (the product passes the CUDA
    kernels, the CPU tests the oracle's); vectors are torch tensors, `p` carries the ghost planes."""

    def __init__(self, layout: SlabLayout, spmv: "SlabSpmv", ops, dist=None, torch=None):
        self.L, self.spmv, self.ops, self.dist, self.torch = layout, spmv, ops, dist, torch

    def _sum(self, v):
        if self.dist is None or self.L.world == 1:
            return v
        # the scalar lives where the vectors live: NCCL reduces CUDA tensors only, gloo (the CPU tests) host tensors
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self._device)
        self.dist.all_reduce(t)  # SUM; the same value on every rank
        return float(t[0])

    def solve(self, b_local, x_local, p_ghosted, r_local, ap_local, max_iterations=500, tolerance=1e-8):
        self._device = getattr(p_ghosted, "device", None)
        """b, x, r, ap: owned rows (n_local); p_ghosted: x_len entries with ghost planes.  Returns
        (iterations, converged, residual_history).  Raises ArithmeticError on a non-finite value (DivergenceError)."""
        if max_iterations < 1 or not tolerance > 0.0:
            raise ValueError("cg_solve: bad configuration")
        L, ops = self.L, self.ops
        p = L.owned(p_ghosted)
        ops.waxpby(0.0, b_local, 0.0, b_local, x_local)   # x = 0
        ops.waxpby(1.0, b_local, 0.0, b_local, r_local)   # r = b
        ops.waxpby(1.0, b_local, 0.0, b_local, p)         # p = b
        bnorm = self._sum(ops.dot(b_local, b_local)) ** 0.5
        rz = self._sum(ops.dot(r_local, r_local))
        history = [1.0]
        if bnorm == 0.0:
            return 0, True, history
        for it in range(1, max_iterations + 1):
            fence = getattr(self.spmv, "fence", None)
            if fence is not None:
                fence()  # neighbours' memory read in place ("p2p"): their update of p is complete
            self.spmv.spmv(p_ghosted, ap_local)
            alpha = rz / self._sum(ops.dot(p, ap_local))
            ops.waxpby(1.0, x_local, alpha, p, x_local)
            ops.waxpby(1.0, r_local, -alpha, ap_local, r_local)
            rr = self._sum(ops.dot(r_local, r_local))
            rz_new = rr
            rel = rr ** 0.5 / bnorm
            history.append(rel)
            if not (alpha == alpha and abs(alpha) != float("inf") and rel == rel and rel != float("inf")):
                raise ArithmeticError(f"non-finite value in iteration {it}")
            if rel <= tolerance:
                return it, True, history
            beta = rz_new / rz
            rz = rz_new
            ops.waxpby(1.0, r_local, beta, p, p)
        return max_iterations, False, history


def build_slab_pattern(sp, layout: SlabLayout, dist=None, diagonal=26.0, off_diagonal=-1.0, perturb=None,
                       values_in_pattern=True, min_pattern_rows=1, stream=None, keep_csr=False):
    """Device-side build of one rank's compressed slab: generate the slab's rows, compress
    them, then merge the per-slab dictionaries over `dist` so every rank holds the GLOBAL
    dictionary and ids numbered as a single-device compression would (first occurrence in
    ascending global row order).  No matrix data crosses ranks -- only the tiny dictionaries.
    `sp` is the paper_1612_00530_b200 package."""
    import numpy as np

    spec = sp.GridSpec(layout.nx, layout.ny, layout.nz_global)
    r0, r1 = layout.row_range
    csr = sp.generate_matrix(spec, diagonal, off_diagonal, perturb=perturb, row_begin=r0, row_end=r1, stream=stream)
    pc = sp.compress_patterns(csr, values_in_pattern, min_pattern_rows=min_pattern_rows, stream=stream)
    if dist is not None and layout.world > 1:
        info = pc.info
        off = pc.download("disp_offsets")
        disp, ends = pc.download("disp_flat"), pc.download("ends_flat")
        first = sp.pattern_first_rows(pc)
        mine = [(int(first[q]) + r0, tuple(disp[off[q]:off[q + 1]].tolist()),
                 tuple(ends[q * info.m:(q + 1) * info.m].tolist())) for q in range(info.n_patterns)]
        table = pc.download("table").tolist()
        gathered = [None] * layout.world
        dist.all_gather_object(gathered, (table, mine))
        if any(t != table for t, _ in gathered):
            raise sp.IntegrityError("slabs disagree on the value table")
        merged, maps = merge_dictionaries([d for _, d in gathered])
        offsets = np.zeros(len(merged) + 1, dtype=np.int64)
        for q, (dd, _) in enumerate(merged):
            offsets[q + 1] = offsets[q] + len(dd)
        flat = np.array([v for dd, _ in merged for v in dd], dtype=np.int32)
        ends_flat = np.array([v for _, ee in merged for v in ee], dtype=np.int32)
        sp.pattern_remap(pc, offsets, flat, ends_flat, np.array(maps[layout.rank], dtype=np.int32), stream=stream)
    return (pc, csr) if keep_csr else pc
