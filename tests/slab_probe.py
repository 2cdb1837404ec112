"""Exploratory: the three kernel calls a middle rank makes per SpMV (interior, lower plane, upper plane) on one GPU."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp
nx = ny = 256; nzl = 256; world = 4; rank = 1
L = sp.SlabLayout(nx, ny, nzl * world, rank, world)
n, plane = L.n_local, L.plane
pc = sp.build_slab_pattern(sp, L, None, keep_csr=False)
x = torch.empty(L.x_len, dtype=torch.float64, device="cuda"); y = torch.empty(n, dtype=torch.float64, device="cuda")
sp.check(sp.lib.spmvb_vec_fill(x.data_ptr(), L.x_len, sp.RANDOM, 7, -1.0, 1.0, L.x_col0, None))
def k(b, e):
    sp.spmv_rows(pc, x, y, b, e, x_col0=L.x_col0, x_len=L.x_len)
def t(fn, reps=50):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
print("x_col0", L.x_col0, "x_len", L.x_len, "n", n)
print(f"whole slab           {t(lambda: k(0, n)):8.1f} us  family {sp.get_option('last_pattern_kernel')}")
print(f"interior planes      {t(lambda: k(plane, n - plane)):8.1f} us  family {sp.get_option('last_pattern_kernel')}")
print(f"lower boundary plane {t(lambda: k(0, plane)):8.1f} us  family {sp.get_option('last_pattern_kernel')}")
print(f"upper boundary plane {t(lambda: k(n - plane, n)):8.1f} us  family {sp.get_option('last_pattern_kernel')}")
for bl in (16, 8, 4, 2):
    sp.set_option("box_lines", bl)
    print(f"lower boundary plane, marches of {bl:2d} lines {t(lambda: k(0, plane)):8.1f} us")
sp.set_option("box_lines", 0)
print(f"all three            {t(lambda: (k(plane, n - plane), k(0, plane), k(n - plane, n))):8.1f} us")

# the streamed driver (no exchange: single process), as bench.py uses it for N > 1
main, comm = torch.cuda.Stream(), torch.cuda.Stream()
class _NoComm:
    P2POp = staticmethod(lambda op, t, peer: None)
    isend = irecv = None
    @staticmethod
    def batch_isend_irecv(ops):
        return []
def ks(xl, yl, b, e, stream=None):
    sp.spmv_rows(pc, xl, yl, b, e, x_col0=L.x_col0, x_len=L.x_len, stream=main if stream is None else stream)
for two in (False, True):
    slab = sp.SlabSpmv(L, ks, _NoComm(), comm, main, torch, two_stream_boundaries=two)
    main.wait_stream(torch.cuda.current_stream())
    for _ in range(3): slab.spmv(x, y)
    main.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(50): slab.spmv(x, y)
    e1.record(main); main.synchronize()
    print(f"SlabSpmv middle rank, boundaries on {'two streams' if two else 'one stream'}: {e0.elapsed_time(e1)/50*1e3:8.1f} us per SpMV (no exchange)")
