"""Exploratory timing of the hybrid (exception-row) path on the GPU box: python tests/hybrid_probe.py [n]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp
n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 128
st = torch.cuda.current_stream()
m = sp.generate_matrix(sp.GridSpec(n1, n1, n1), perturb=(11, 0.1, 0.1))
pc = sp.compress_patterns(m, True, min_pattern_rows=2)
info = pc.info
n = info.n
print("rows", n, "patterns", info.n_patterns, "exceptions", info.n_exc, "w_exc", info.w_exc, "plan", info.kernel_plan)
alg = 20.0 * n + info.n_exc * (4.0 + 12.0 * info.w_exc)
ell = sp.to_ell(m, min_width=27)
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
y2 = torch.empty(n, dtype=torch.float64, device="cuda")
sp.check(sp.lib.spmvb_vec_fill(x.data_ptr(), n, sp.RANDOM, 7, -1.0, 1.0, 0, None))
# reference bits: List 1 for the dictionary rows, the ELL kernel with a row map for the exception rows
sp.set_option("pattern_kernel", 1); sp.set_option("exception_kernel", 1)
sp.spmv_rows(pc, x, y2, 0, n)
sp.set_option("pattern_kernel", 0); sp.set_option("exception_kernel", 0)
torch.cuda.synchronize()
def timeit(a, label, reps=100, **opts):
    for k, v in opts.items():
        sp.set_option(k, v)
    y.fill_(float("nan"))
    for _ in range(3):
        sp.spmv_rows(a, x, y, 0, n)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sp.spmv_rows(a, x, y, 0, n)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e3
    g = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        with torch.cuda.graph(g, stream=s2):
            for _ in range(20):
                sp.spmv_rows(a, x, y, 0, n, stream=s2)
        g.replay(); s2.synchronize()
        e0.record(s2)
        for _ in range(5):
            g.replay()
        e1.record(s2); s2.synchronize()
    tg = e0.elapsed_time(e1) / 100 * 1e3
    bad = int((y.view(torch.int64) != y2.view(torch.int64)).sum()) if a is pc else -1
    print(f"{label:44s} {t:8.1f} us (graph replay {tg:7.1f} us)  frac of 6544 GB/s {alg / min(t, tg) / 1e3 / 6544:.3f}  family {sp.get_option('last_pattern_kernel')}  rows differing {bad}")
    for k in opts:
        sp.set_option(k, 1 if k == "exception_overlap" else 0)
timeit(pc, "hybrid default (ring + ELL kernel, row map)")
timeit(pc, "hybrid, one kernel after the other", exception_overlap=0)
timeit(pc, "hybrid windows, 64-row tiles", exception_kernel=64)
timeit(pc, "hybrid windows, 32-row tiles", exception_kernel=32)
timeit(pc, "hybrid List 1 kernel + default block", pattern_kernel=1)
timeit(ell, "uncompressed ELL")
