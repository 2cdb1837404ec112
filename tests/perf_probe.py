"""Exploratory kernel timing on the GPU box (not a test, not the bench):
python tests/perf_probe.py [n] [reps].  Formats are built by the oracle here
only because this probe predates the device builders; bench.py does not do that."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp  # noqa: E402
from oracle import oracle as orc  # noqa: E402

dims = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128").split("x")]
g = tuple(dims * 3) if len(dims) == 1 else tuple(dims)
n1 = g[0]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
fmts = sys.argv[3].split(",") if len(sys.argv) > 3 else ["pattern", "generic", "vt", "ell"]
n = g[0] * g[1] * g[2]
ring_lines = [int(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else []
only_ring = bool(ring_lines)
nnz = (3 * g[0] - 2) * (3 * g[1] - 2) * (3 * g[2] - 2)
print("grid", g, "rows", n, flush=True)
t0 = time.time()
pc = orc.compress_patterns_grid(*g, values_in_pattern=True)
print(f"oracle pattern build {time.time()-t0:.1f}s", flush=True)
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
sp.lib.spmvb_vec_fill(x.data_ptr(), n, 2, 7, -1.0, 1.0, 0, None)
torch.cuda.synchronize()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def timeit(a, label, bytes_per_row, **opts):
    for k, v in opts.items():
        sp.set_option(k, v)
    st = torch.cuda.current_stream()
    for _ in range(3):
        sp.spmv_rows(a, x, y, 0, n, stream=st)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for s, e in ev:
        flush.zero_()
        s.record()
        sp.spmv_rows(a, x, y, 0, n, stream=st)
        e.record()
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) * 1e3 for s, e in ev)
    med = ts[len(ts) // 2]
    # back-to-back (no flush) average
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        sp.spmv_rows(a, x, y, 0, n, stream=st)
    e.record()
    torch.cuda.synchronize()
    b2b = s.elapsed_time(e) * 1e3 / reps
    print(f"{label:34s} flushed med {med:9.1f} us  min {ts[0]:9.1f} | b2b {b2b:9.1f} us ({b2b * 1e3 / n:6.3f} ns/krow) "
          f"{2*nnz/b2b/1e3:9.1f} GF/s  {bytes_per_row*n/b2b/1e3:8.1f} GB/s ({bytes_per_row} B/row)", flush=True)
    for k in opts:
        sp.set_option(k, 0 if k != "box_prefetch" else -1)


if "pattern" in fmts or "generic" in fmts:
    d = sp.upload_pattern(pc.n, pc.table, pc.disp_offsets, pc.disp_flat, pc.ends_flat, pc.row_pattern, True)
    ref = None
    if "pattern" in fmts:
        for march, name in ((0, "default (tensor ring)"), (3, "sliding window box3 <8,4,2,1,3>"), (1, "box3 R=16"), (5, "box3 Q=1 2 lines/step"),
                            (12, "box3 full-line CTA"), (70, "box3 look-ahead 1"), (20, "box5 cp.async ring"), (35, "box6 4 cols/thread"),
                            (30, "box6 8 cols/thread"), (47, "box7 pipelined ring"), (62, "box8 TMA ring 8w R=8"),
                            (101, "ring: chunk per warp"), (108, "ring: round-robin tiles per CTA"), (109, "ring: round-robin tiles per warp"),
                            (104, "ring: 2 planes/thread, 6 slots"), (110, "ring: 4 planes/thread 12w, chunk/CTA"), (115, "ring: 6 planes, rr tiles/CTA"), (116, "ring: 6 planes, chunk/warp"), (117, "ring: 6 planes, rr tiles/warp"), (107, "ring: 5 slots, ids by loads"), (96, "ring: + TMA L2 prefetch 2"),
                            (105, "ring: st.cs stores"), (97, "ABLATION (chunk/warp) no FP chains"),
                            (98, "ABLATION (chunk/warp) one LDS quad/step"), (99, "ABLATION (chunk/warp) fetch+store only"),
                            (100, "ABLATION (chunk/warp) fetch only"), (103, "ABLATION fetch+store only"), (102, "ABLATION fetch only"),
                            (106, "ABLATION fetch only, no left-over column"), (118, "ABLATION default, no left-over column (wrong col)"),
                            (119, "ABLATION default, fetch+store only"), (120, "ABLATION default, fetch only")):
            if march >= 90 and ring_lines:
                for ln in ring_lines:
                    timeit(d, f"pattern {name} R={ln}", 20, pattern_kernel=2, box_march=march, box_prefetch=2, box_lines=ln)
                continue
            if only_ring and march not in (0,):
                continue
            timeit(d, f"pattern {name}", 20, pattern_kernel=2, box_march=march, box_prefetch=2)
        timeit(d, "pattern box v2 <16,8,2,0> pf=4", 20, pattern_kernel=3, box_march=0, box_prefetch=4)
    if "generic" in fmts:
        timeit(d, "pattern generic", 20, pattern_kernel=1)
    del d
if "vt" in fmts or "ell" in fmts:
    t0 = time.time()
    m = orc.generate_matrix(*g)
    print(f"oracle csr build {time.time()-t0:.1f}s", flush=True)
    if "vt" in fmts:
        vt = orc.compress_values(m)
        d = sp.upload_vt(vt.n, vt.width, vt.table, vt.sorted_columns, vt.ends)
        del vt
        timeit(d, "vt staged vector loads", 132)
        timeit(d, "vt tma pipeline", 132, ell_kernel=3)
        del d
    if "ell" in fmts:
        e = orc.to_ell(m)
        d = sp.upload_ell(e.n, e.width, e.nnz, e.values, e.columns)
        del e
        timeit(d, "ell tma pipeline", 340)
        timeit(d, "ell staged vector loads", 340, ell_kernel=2)
        timeit(d, "ell naive", 340, ell_kernel=1)
