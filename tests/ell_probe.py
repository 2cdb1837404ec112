"""Exploratory: ELL / vt kernel variants at 256^3 (GPU box): python tests/ell_probe.py"""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp
n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = sp.GridSpec(n1, n1, n1)
m = sp.generate_matrix(g); n = m.n
ell = sp.to_ell(m, min_width=27); vt = sp.compress_values(m, min_width=27)
x = sp.DeviceVector(n); y = sp.DeviceVector(n); ref = sp.DeviceVector(n)
sp.check(sp.lib.spmvb_vec_fill(sp.C.c_void_p(x.ptr), n, 2, 7, -1.0, 1.0, 0, None))
def timed(a, reps=20):
    sp.spmv_rows(a, x, y, 0, n); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): sp.spmv_rows(a, x, y, 0, n)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
sp.set_option("ell_kernel", 2); sp.spmv_rows(ell, x, ref, 0, n)
for name, a, bpr, ks in (("ell", ell, 340, (0, 2, 3, 4, 5, 6)), ("vt", vt, 132, (0, 2, 3, 6, 7))):
    for k in ks:
        sp.set_option("ell_kernel", k)
        ms = timed(a)
        same = sp.compare(y, ref, n)[1] == 0 if name == "ell" else None
        print(f"{name} ell_kernel={k}: {ms*1e3:8.1f} us  {bpr*n/ms/1e6:8.1f} GB/s  bit-identical to the staged kernel: {same}")
sp.set_option("ell_kernel", 0)
