"""Scratch: one tensor-ring launch on a small grid (used under compute-sanitizer)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp
from oracle import oracle as orc
g = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128x12x10").split("x"))
march = int(sys.argv[2]) if len(sys.argv) > 2 else 90
m = orc.generate_matrix(*g)
pc = orc.compress_patterns(m, True)
d = sp.upload_pattern(pc.n, pc.table, pc.disp_offsets, pc.disp_flat, pc.ends_flat, pc.row_pattern, True)
x = orc.make_test_vector(m.n, orc.RANDOM, seed=5, lo=-1.0, hi=1.0)
sp.set_option("box_march", march)
y = sp.spmv(d, x)
print("kernel family", sp.get_option("last_pattern_kernel"))
ref = orc.spmv(pc, x)
bad = np.flatnonzero(y.view(np.uint64) != ref.view(np.uint64))
print("rows differing:", bad.size, bad[:20])
