"""Multi-slab SpMV on ONE GPU: the z-slab driver (SlabSpmv), the device-side slab build and
the dictionary merge, with the halo exchange emulated by device copies between the slabs'
ghosted vectors.  (One process per GPU over NCCL is the real deployment; only one GPU is
available to the tests, and ranks that wait on each other must not be emulated as
concurrent kernels, so the slabs run one after the other here.)"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class _LocalExchange:
    """Stands in for torch.distributed between slabs that live in one process: isend/irecv
    become device copies between the registered per-rank x_local tensors."""

    class P2POp:
        def __init__(self, op, tensor, peer):
            self.op, self.tensor, self.peer = op, tensor, peer

    isend, irecv = "isend", "irecv"

    def __init__(self):
        self.sends = {}

    def batch_isend_irecv(self, ops):
        for o in ops:
            if o.op == "isend":
                self.sends[(o.rank_from, o.peer, o.tag)] = o.tensor
        return []


def test_two_and_three_slabs_equal_the_whole_matrix(orc):
    import torch

    import paper_1612_00530_b200 as sp

    for (nx, ny, nz), world in (((64, 12, 10), 2), ((128, 10, 9), 3), ((256, 8, 8), 2)):
        plane = nx * ny
        whole = orc.compress_patterns_grid(nx, ny, nz, values_in_pattern=True)
        xg = orc.make_test_vector(nx * ny * nz, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
        ref = orc.spmv(whole, xg)
        layouts = [sp.SlabLayout(nx, ny, nz, r, world) for r in range(world)]
        # device-side slab build + dictionary merge (same arithmetic as build_slab_pattern over torch.distributed)
        slabs, dicts = [], []
        for L in layouts:
            r0, r1 = L.row_range
            csr = sp.generate_matrix(sp.GridSpec(nx, ny, nz), row_begin=r0, row_end=r1)
            pc = sp.compress_patterns(csr, True)
            info, off = pc.info, pc.download("disp_offsets")
            disp, ends, first = pc.download("disp_flat"), pc.download("ends_flat"), sp.pattern_first_rows(pc)
            dicts.append([(int(first[q]) + r0, tuple(disp[off[q]:off[q + 1]].tolist()),
                           tuple(ends[q * info.m:(q + 1) * info.m].tolist())) for q in range(info.n_patterns)])
            slabs.append(pc)
        merged, maps = sp.merge_dictionaries(dicts)
        offsets = np.zeros(len(merged) + 1, dtype=np.int64)
        for q, (dd, _) in enumerate(merged):
            offsets[q + 1] = offsets[q] + len(dd)
        flat = np.array([v for dd, _ in merged for v in dd], dtype=np.int32)
        ends_flat = np.array([v for _, ee in merged for v in ee], dtype=np.int32)
        for L, pc, mp in zip(layouts, slabs, maps):
            sp.pattern_remap(pc, offsets, flat, ends_flat, np.array(mp, dtype=np.int32))
            r0, r1 = L.row_range
            # after the merge every slab's ids are the slice of the single-matrix compression
            assert np.array_equal(pc.download("row_pattern"), whole.row_pattern[r0:r1])
            assert np.array_equal(pc.download("disp_flat"), whole.disp_flat)
        # ghosted local vectors: owned part filled on the device, ghosts poisoned
        xs = []
        for L in layouts:
            x = torch.full((L.x_len,), float("nan"), dtype=torch.float64, device="cuda")
            sp.check(sp.lib.spmvb_vec_fill(L.owned(x).data_ptr(), L.n_local, sp.RANDOM, 7, -1.0, 1.0, L.row_range[0], None))
            if not L.has_lower:
                x[:plane] = 0.0
            if not L.has_upper:
                x[plane + L.n_local:] = 0.0
            xs.append(x)
        # the exchange SlabSpmv would post: first/last owned plane -> neighbours' ghosts
        for r, L in enumerate(layouts):
            if L.has_lower:
                xs[r - 1][plane + layouts[r - 1].n_local:] = xs[r][plane:2 * plane]
            if L.has_upper:
                xs[r + 1][:plane] = xs[r][L.n_local:L.n_local + plane]
        torch.cuda.synchronize()
        for r, (L, pc) in enumerate(zip(layouts, slabs)):
            y = torch.full((L.n_local,), float("nan"), dtype=torch.float64, device="cuda")
            calls = []

            def kernel(xl, yl, b, e, pc=pc, L=L):
                calls.append((b, e))
                sp.spmv_rows(pc, xl, yl, b, e, x_col0=L.x_col0, x_len=L.x_len)

            class _NoComm:  # exchange already done above; SlabSpmv still splits interior / boundary planes
                P2POp = staticmethod(lambda op, t, peer: None)
                isend = irecv = None

                @staticmethod
                def batch_isend_irecv(ops):
                    return []

            sp.SlabSpmv(L, kernel, _NoComm()).spmv(xs[r], y)
            torch.cuda.synchronize()
            r0, r1 = L.row_range
            assert np.array_equal(y.cpu().numpy().view(np.uint64), ref[r0:r1].view(np.uint64)), (nx, ny, nz, world, r)
            assert len(calls) == (1 if world == 1 else 1 + int(L.has_lower) + int(L.has_upper))
            # the streamed form bench.py uses: exchange on a side stream, the two boundary planes on two streams
            main, comm = torch.cuda.Stream(), torch.cuda.Stream()
            y2 = torch.full((L.n_local,), float("nan"), dtype=torch.float64, device="cuda")
            streams_used = []

            def kernel_s(xl, yl, b, e, stream=None, pc=pc, L=L):
                streams_used.append(comm if stream is comm else main)
                sp.spmv_rows(pc, xl, yl, b, e, x_col0=L.x_col0, x_len=L.x_len, stream=main if stream is None else stream)

            main.wait_stream(torch.cuda.current_stream())
            sp.SlabSpmv(L, kernel_s, _NoComm(), comm, main, torch, two_stream_boundaries=True).spmv(xs[r], y2)
            main.synchronize()
            assert np.array_equal(y2.cpu().numpy().view(np.uint64), ref[r0:r1].view(np.uint64)), (nx, ny, nz, world, r)
            if L.has_lower and L.has_upper:
                assert comm in streams_used and main in streams_used
