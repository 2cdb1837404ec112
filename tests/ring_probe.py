"""Exploratory timing of the default pattern kernel on the GPU box (not a test, not the bench):
python tests/ring_probe.py [grid ...] [key=value ...]   e.g.  256 128 512x512x64 box_march=110
Device-side build; back-to-back launches on one stream (CUDA events) and a check of y against the List-1 kernel."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp  # noqa: E402

grids, opts = [], {}
for a in sys.argv[1:]:
    if "=" in a:
        k, v = a.split("=")
        opts[k] = int(v)
    else:
        d = [int(v) for v in a.split("x")]
        grids.append(tuple(d * 3) if len(d) == 1 else tuple(d))
if not grids:
    grids = [(256, 256, 256)]
st = torch.cuda.Stream()
reps = 200
with torch.cuda.stream(st):
    for g in grids:
        n = g[0] * g[1] * g[2]
        nnz = (3 * g[0] - 2) * (3 * g[1] - 2) * (3 * g[2] - 2)
        pc = sp.compress_patterns(sp.generate_matrix(sp.GridSpec(*g), stream=st), True, stream=st)
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        y2 = torch.empty(n, dtype=torch.float64, device="cuda")
        sp.check(sp.lib.spmvb_vec_fill(x.data_ptr(), n, sp.RANDOM, 7, -1.0, 1.0, 0, st.cuda_stream))
        sp.set_option("pattern_kernel", 1)
        sp.spmv_rows(pc, x, y2, 0, n, stream=st)
        sp.set_option("pattern_kernel", 0)
        for k, v in opts.items():
            sp.set_option(k, v)
        y.fill_(float("nan"))
        for _ in range(5):
            sp.spmv_rows(pc, x, y, 0, n, stream=st)
        fam = sp.get_option("last_pattern_kernel")
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                sp.spmv_rows(pc, x, y, 0, n, stream=st)
            e1.record(st)
            st.synchronize()
            best = min(best, e0.elapsed_time(e1) / reps * 1e3)
        bad = int((y.view(torch.int64) != y2.view(torch.int64)).sum())
        # the same launches replayed from a CUDA graph: host launch cost leaves the measurement (small grids)
        gtime = float("nan")
        try:
            g_ = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_, stream=st):
                for _ in range(50):
                    sp.spmv_rows(pc, x, y, 0, n, stream=st)
            g_.replay()
            st.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(4):
                g_.replay()
            e1.record(st)
            st.synchronize()
            gtime = e0.elapsed_time(e1) / 200 * 1e3
            del g_
        except Exception as ex:  # noqa: BLE001
            print("graph capture failed:", ex)
        for k in opts:
            sp.set_option(k, 0)
        print(f"grid {g}: {best:8.2f} us (graph replay {gtime:7.2f} us)  {20.0 * n / best / 1e3:7.1f} GB/s ({20.0 * n / best / 1e3 / 6544:.3f} of 6544)  "
              f"{2 * nnz / best / 1e3:8.1f} GF/s  family {fam}  rows differing from List 1: {bad}  opts {opts}", flush=True)
        del pc, x, y, y2
