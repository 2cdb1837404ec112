"""Exploratory: where the time of a CG solve goes (GPU box): python tests/cg_diag.py [n]"""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp
n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 256
m = sp.generate_matrix(sp.GridSpec(n1, n1, n1))
n = m.n
ones = sp.DeviceVector(n); b = sp.DeviceVector(n)
sp.check(sp.lib.spmvb_vec_fill(sp.C.c_void_p(ones.ptr), n, 0, 0, 0.0, 1.0, 0, None))
ell = sp.to_ell(m, min_width=27)
sp.spmv_rows(ell, ones, b, 0, n)
a = sp.compress_patterns(m, True)
for its in (1, 1, 2, 5, 10, 30, 60, 60):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = sp.cg_solve(a, b, max_iterations=its, tolerance=1e-30)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"its {its:3d}: {dt*1e3:9.3f} ms total, {dt/rep.iterations*1e6:9.1f} us/iteration, kernel {sp.get_option('last_pattern_kernel')}")
y = sp.DeviceVector(n)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(20): sp.spmv_rows(a, ones, y, 0, n)
    torch.cuda.synchronize(); print(f"spmv x20: {(time.perf_counter()-t0)/20*1e6:.1f} us each")
# with the other handles alive (as cg_probe has them): repeated solves and raw allocation timings
vt = sp.compress_values(m, min_width=27)
torch.cuda.synchronize()
for rep in range(8):
    t0 = time.perf_counter()
    x, r = sp.cg_solve(a, b, max_iterations=60, tolerance=1e-30)
    torch.cuda.synchronize()
    print(f"solve {rep}: {(time.perf_counter()-t0)*1e3:9.3f} ms")
for rep in range(8):
    t0 = time.perf_counter()
    vs = [sp.DeviceVector(n) for _ in range(3)]
    t1 = time.perf_counter()
    del vs
    torch.cuda.synchronize()
    print(f"alloc x3 {(t1-t0)*1e3:8.3f} ms   free x3 {(time.perf_counter()-t1)*1e3:8.3f} ms")
