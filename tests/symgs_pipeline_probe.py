"""Exploratory (GPU box): the pipelined symgs sweep against the per-level kernel -- bits and time.
python tests/symgs_pipeline_probe.py [grid ...]"""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp

grids = []
for a in sys.argv[1:]:
    d = [int(v) for v in a.split("x")]
    grids.append(tuple(d * 3) if len(d) == 1 else tuple(d))
if not grids:
    grids = [(3, 3, 1), (5, 4, 3), (33, 7, 9), (40, 30, 20), (64, 64, 64), (100, 256, 7), (128, 128, 128), (256, 256, 256)]
for gr in grids:
    g = sp.GridSpec(*gr)
    m = sp.generate_matrix(g); n = m.n
    x = sp.DeviceVector(n); b = sp.DeviceVector(n)
    sp.check(sp.lib.spmvb_vec_fill(sp.C.c_void_p(b.ptr), n, sp.RANDOM, 5, -1.0, 1.0, 0, None))
    ref = None
    for pipe, pers, lag in ((0, 0, 0), (0, 1, 0), (1, 1, 0), (1, 1, 8)):
        sp.set_option("symgs_pipeline", pipe); sp.set_option("symgs_persistent", pers); sp.set_option("symgs_lag", lag)
        sp.check(sp.lib.spmvb_vec_fill(sp.C.c_void_p(x.ptr), n, sp.RANDOM, 9, -1.0, 1.0, 0, None))
        sp.symgs_sweep(m, g, x, b); sp.symgs_sweep(m, g, x, b); torch.cuda.synchronize()
        y = x.to_host()
        if ref is None: ref = y
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps): sp.symgs_sweep(m, g, x, b)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps * 1e3
        bad = int((y.view(np.uint64) != ref.view(np.uint64)).sum())
        print(f"{gr} pipeline {pipe} persistent {pers} lag {lag}: {dt:8.3f} ms per sweep, rows differing from the level kernel: {bad}", flush=True)
    sp.set_option("symgs_pipeline", 1); sp.set_option("symgs_persistent", 1); sp.set_option("symgs_lag", 0)
