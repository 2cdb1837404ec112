"""Run a few vt / ELL launches at n^3 (for ncu): python tests/prof_vt.py n fmt"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp
n1 = int(sys.argv[1]); fmt = sys.argv[2]
m = sp.generate_matrix(sp.GridSpec(n1, n1, n1))
a = sp.compress_values(m, min_width=27) if fmt == "vt" else sp.to_ell(m, min_width=27)
n = m.n
del m
x = torch.empty(n, dtype=torch.float64, device="cuda"); y = torch.empty(n, dtype=torch.float64, device="cuda")
sp.check(sp.lib.spmvb_vec_fill(x.data_ptr(), n, 2, 7, -1.0, 1.0, 0, None))
for _ in range(4):
    sp.spmv_rows(a, x, y, 0, n)
torch.cuda.synchronize()
print("ok")
