"""Exploratory: time of one symgs sweep on the device, direct launches vs the recorded graph (GPU box): python tests/symgs_probe.py"""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp
for n1 in (64, 128, 256):
    g = sp.GridSpec(n1, n1, n1)
    m = sp.generate_matrix(g); n = m.n
    x = sp.DeviceVector(n); b = sp.DeviceVector(n)
    sp.check(sp.lib.spmvb_vec_fill(sp.C.c_void_p(b.ptr), n, 0, 0, 0.0, 1.0, 0, None))
    for graph in (0, 1, 2):
        sp.set_option("symgs_persistent", 1 if graph == 2 else 0)
        sp.set_option("symgs_graph", min(graph, 1))
        sp.check(sp.lib.spmvb_vec_fill(sp.C.c_void_p(x.ptr), n, 0, 0, 0.0, 0.0, 0, None))
        torch.cuda.synchronize(); t0 = time.perf_counter()
        sp.symgs_sweep(m, g, x, b); torch.cuda.synchronize()
        first = time.perf_counter() - t0
        t0 = time.perf_counter()
        for _ in range(5): sp.symgs_sweep(m, g, x, b)
        torch.cuda.synchronize()
        levels = 7 * (n1 - 1) + 1
        print(f"{n1}^3 {('direct launches', 'graph of launches', 'persistent kernel')[graph]}: first sweep {first*1e3:8.2f} ms, then {(time.perf_counter()-t0)/5*1e3:8.2f} ms per sweep ({2*levels} launches)")
    a = sp.compress_patterns(m, True)
    ones = sp.DeviceVector(n); rhs = sp.DeviceVector(n)
    sp.check(sp.lib.spmvb_vec_fill(sp.C.c_void_p(ones.ptr), n, 0, 0, 0.0, 1.0, 0, None))
    sp.spmv_rows(a, ones, rhs, 0, n)
    for sweeps in (0, 1):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        xs, rep = sp.cg_solve(a, rhs, tolerance=1e-8, symgs_sweeps=sweeps, csr=m, grid=g)
        torch.cuda.synchronize()
        print(f"{n1}^3 cg symgs_sweeps={sweeps}: {rep.iterations} iterations, {(time.perf_counter()-t0)*1e3:.1f} ms, converged {rep.converged}")
