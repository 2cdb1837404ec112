"""Exploratory: time per CG iteration on the device (GPU box): python tests/cg_probe.py [n]"""
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
for name, a in (("pattern", sp.compress_patterns(m, True)), ("vt", sp.compress_values(m, min_width=27)), ("ell", ell)):
    x, rep = sp.cg_solve(a, b, max_iterations=30, tolerance=1e-30)
    sol = x  # reused for every solve below: nothing is allocated or freed inside the timed calls
    times = []
    for _ in range(7):  # a solve is host-driven: report the median, and the spread (a shared box stalls now and then)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = sp.cg_solve(a, b, max_iterations=60, tolerance=1e-30, x=sol)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) / rep.iterations * 1e6)
    times.sort()
    print(f"{name:8s} {n1}^3: {times[3]:8.1f} us per CG iteration, median of 7 solves of {rep.iterations} iterations "
          f"(min {times[0]:.1f}, max {times[-1]:.1f}; residual {rep.residual_history[-1]:.2e})")
