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
ell = sp.to_ell(m, min_width=27)
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
y2 = torch.empty(n, dtype=torch.float64, device="cuda")
sp.check(sp.lib.spmvb_vec_fill(x.data_ptr(), n, sp.RANDOM, 7, -1.0, 1.0, 0, None))
def timeit(a, label, reps=50, **opts):
    for k, v in opts.items():
        sp.set_option(k, v)
    for _ in range(3):
        sp.spmv_rows(a, x, y, 0, n)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sp.spmv_rows(a, x, y, 0, n)
    e1.record()
    torch.cuda.synchronize()
    print(f"{label:40s} {e0.elapsed_time(e1) / reps * 1e3:9.1f} us  family {sp.get_option('last_pattern_kernel')}")
    for k in opts:
        sp.set_option(k, 0)
timeit(pc, "hybrid default")
sp.spmv_rows(pc, x, y2, 0, n)
torch.cuda.synchronize()
timeit(pc, "hybrid sliding window (box3)", box_march=3)
print("bit differences ring vs box3:", int((y.view(torch.int64) != y2.view(torch.int64)).sum()))
timeit(pc, "hybrid List 1 kernel", pattern_kernel=1)
print("bit differences list1 vs ring:", int((y.view(torch.int64) != y2.view(torch.int64)).sum()))
timeit(ell, "uncompressed ELL")
