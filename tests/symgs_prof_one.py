"""One symgs sweep at 128^3 (for ncu): python tests/symgs_prof_one.py [n]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp
n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 128
g = sp.GridSpec(n1, n1, n1)
m = sp.generate_matrix(g)
x = sp.DeviceVector(m.n); b = sp.DeviceVector(m.n)
sp.check(sp.lib.spmvb_vec_fill(sp.C.c_void_p(b.ptr), m.n, sp.RANDOM, 5, -1.0, 1.0, 0, None))
sp.check(sp.lib.spmvb_vec_fill(sp.C.c_void_p(x.ptr), m.n, sp.RANDOM, 9, -1.0, 1.0, 0, None))
for _ in range(3):
    sp.symgs_sweep(m, g, x, b)
torch.cuda.synchronize()
print("kernel", sp.get_option("last_symgs_kernel"))
