"""Exploratory: what the z-slab decomposition costs on ONE device (spmvb_multi_*, logical slabs, same-device ghost copies).
G slabs of nx x ny x nzl each run back to back; time per slab = total / G, against the undivided slab."""
import sys
sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp

nx = ny = int(sys.argv[1]) if len(sys.argv) > 1 else 256
nzl = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = 100
print(f"grid {nx}x{ny}, {nzl} planes per slab")
for G in (1, 2, 4):
    ms = sp.MultiSlab(sp.GridSpec(nx, ny, nzl * G), [0] * G)
    ms.fill_x(sp.RANDOM, 7, -1.0, 1.0)
    for mode, name in ((sp.SLAB_SERIAL, "serial (copies, one launch)"), (sp.SLAB_OVERLAP, "overlap (copies || interior, 2 planes)")):
        for graph in (1, 0):
            sp.set_option("slab_graph", graph)
            wall, dev = ms.bench(reps, mode)
            print(f"G={G} {name:40s} graph={graph}: device {dev / reps / G * 1e6:7.1f} us per slab-SpMV, host wall {wall / reps / G * 1e6:7.1f} us")
    sp.set_option("slab_graph", 1)
    del ms

# One slab alone, as a GPU of a multi-GPU run sees it: the middle slab of three, ghost copies from its neighbours' planes
# (same-device copies here, peer copies over NVLink there), everything on one stream.
import ctypes as C
ms = sp.MultiSlab(sp.GridSpec(nx, ny, nzl * 3), [0] * 3)
ms.fill_x(sp.RANDOM, 7, -1.0, 1.0)
parts = [ms.part(g) for g in range(3)]
_, z0, z1, a, xg, yg = parts[1]
plane = nx * ny
n = (z1 - z0) * plane
lo_src = parts[0][4].ptr + 8 * (parts[0][2] - parts[0][1]) * plane   # the lower neighbour's last owned plane
hi_src = parts[2][4].ptr + 8 * plane                                # the upper neighbour's first owned plane
slab = sp.Slab(a, plane, True, True)
import torch
st = torch.cuda.Stream()
def timed(fn, reps=200):
    for _ in range(5): fn()
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps): fn()
    e1.record(st); st.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
t_whole = timed(lambda: sp.spmv_rows(a, xg, yg, 0, n, x_col0=(z0 - 1) * plane, x_len=n + 2 * plane, stream=st))
print(f"middle slab, all rows in one launch, no exchange:        {t_whole:7.1f} us")
for mode, name in ((sp.SLAB_SERIAL, "serial"), (sp.SLAB_OVERLAP, "overlap")):
    for graph in (1, 0):
        sp.set_option("slab_graph", graph)
        t = timed(lambda: slab.spmv(xg, yg, lo_src, hi_src, mode, stream=st))
        print(f"middle slab, spmvb_slab_spmv {name:8s} graph={graph} (2 ghost copies + launches): {t:7.1f} us  (+{t - t_whole:.1f})")
sp.set_option("slab_graph", 1)
