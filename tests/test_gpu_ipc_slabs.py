"""Two processes on ONE device, each the rank of a z-slab run with the "p2p" exchange: every rank maps its neighbour's
vector through CUDA IPC (spmvb_ipc_*) and spmvb_slab_spmv pulls the boundary planes in front of its single launch, replayed
as a CUDA graph -- the code path bench.py --exchange p2p runs on a multi-GPU box, minus NVLink.  gloo carries the control
plane (dictionary merge, barriers, CG's all-reduces of host scalars).  No kernel waits on another rank's kernel."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["SPMVB_ROOT"])
import paper_1612_00530_b200 as sp
from oracle import oracle as orc

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(0)
sp.check(sp.lib.spmvb_set_device(0))
g = (128, 12, 16)
nx, ny, nz = g
L = sp.SlabLayout(nx, ny, nz, rank, world)
r0, r1 = L.row_range
n = L.n_local
main, comm = torch.cuda.Stream(), torch.cuda.Stream()
whole = orc.compress_patterns_grid(*g, values_in_pattern=True)
xg = orc.make_test_vector(whole.n, orc.RANDOM, seed=7, lo=-1.0, hi=1.0)
bits = lambda a: np.ascontiguousarray(a).view(np.uint64)
with torch.cuda.stream(main):
    pc = sp.build_slab_pattern(sp, L, dist, stream=main)
    assert np.array_equal(pc.download("row_pattern"), whole.row_pattern[r0:r1])  # ids after the dictionary merge
    xv = sp.DeviceVector(L.x_len)  # cudaMalloc'ed: exportable
    x = torch.as_tensor(xv, device="cuda")
    x.fill_(float("nan"))  # ghosts poisoned until the exchange fills them
    L.owned(x).copy_(torch.from_numpy(xg[r0:r1]))
    y = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    main.synchronize()
    for schedule in ("serial", "overlap"):
        slab = sp.DeviceSlabSpmv(sp, L, pc, dist, main, comm, torch, exchange="p2p", schedule=schedule)
        slab.fence()
        used = []
        for _ in range(4):  # direct launches, graph capture, two replays
            y.fill_(float("nan"))
            slab.spmv(x, y)
            used.append(slab.slab.last_was_graph)
        main.synchronize()
        assert used == [False, True, True, True], used
        ref = orc.spmv(whole, xg)[r0:r1]
        assert np.array_equal(bits(y.cpu().numpy()), bits(ref)), f"rank {rank} {schedule}"
        dist.barrier()  # nobody unmaps while a neighbour may still pull
        slab.unmap_neighbours()

    # distributed CG over the two slabs: the search direction changes every iteration, the exchange is real
    class Ops:
        @staticmethod
        def dot(u, v):
            out = sp.C.c_double()
            sp.check(sp.lib.spmvb_dot(sp.C.c_void_p(u.data_ptr()), sp.C.c_void_p(v.data_ptr()), u.numel(), sp.C.byref(out), main.cuda_stream))
            return out.value

        @staticmethod
        def waxpby(alpha, xx, beta, yy, w):
            sp.check(sp.lib.spmvb_waxpby(alpha, sp.C.c_void_p(xx.data_ptr()), beta, sp.C.c_void_p(yy.data_ptr()),
                                         sp.C.c_void_p(w.data_ptr()), xx.numel(), main.cuda_stream))

    xs = orc.make_test_vector(whole.n, orc.RANDOM, seed=3, lo=-1.0, hi=1.0)
    b = orc.spmv(whole, xs)
    pv = sp.DeviceVector(L.x_len)
    p_g = torch.as_tensor(pv, device="cuda")
    p_g.zero_()
    z = lambda k: torch.zeros(k, dtype=torch.float64, device="cuda")
    b_d, x_d, r_d, ap_d = torch.from_numpy(np.ascontiguousarray(b[r0:r1])).cuda(), z(n), z(n), z(n)
    slab = sp.DeviceSlabSpmv(sp, L, pc, dist, main, comm, torch, exchange="p2p", schedule="serial")
    class HostSum(sp.SlabCg):  # gloo reduces host tensors: the scalars of the dots
        def _sum(self, v):
            t = torch.tensor([v], dtype=torch.float64)
            dist.all_reduce(t)
            return float(t[0])
    cg = HostSum(L, slab, Ops, dist, torch)
    it, conv, hist = cg.solve(b_d, x_d, p_g, r_d, ap_d, max_iterations=300, tolerance=1e-10)
    main.synchronize()
    assert conv and np.abs(x_d.cpu().numpy() - xs[r0:r1]).max() <= 1e-7, (it, conv)
    its = [None] * world
    dist.all_gather_object(its, it)
    assert its[0] == its[1]
    dist.barrier()
    slab.unmap_neighbours()
print(f"rank {rank} ok iterations {it}")
dist.destroy_process_group()
'''


def test_two_ranks_on_one_device_exchange_through_cuda_ipc(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SPMVB_ROOT=ROOT)
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out)
    for rank, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0 and f"rank {rank} ok" in out, out[-3000:]
