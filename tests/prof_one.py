"""Run a few launches of one pattern-kernel configuration (for ncu).
python tests/prof_one.py n march pf reps [kernel]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp  # noqa: E402
from oracle import oracle as orc  # noqa: E402

n1, march, pf, reps = (int(v) for v in sys.argv[1:5])
kernel = int(sys.argv[5]) if len(sys.argv) > 5 else 2
pc = orc.compress_patterns_grid(n1, n1, n1, values_in_pattern=True)
n = pc.n
d = sp.upload_pattern(pc.n, pc.table, pc.disp_offsets, pc.disp_flat, pc.ends_flat, pc.row_pattern, True)
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
sp.lib.spmvb_vec_fill(x.data_ptr(), n, 2, 7, -1.0, 1.0, 0, None)
sp.set_option("pattern_kernel", kernel)
sp.set_option("box_march", march)
sp.set_option("box_prefetch", pf)
torch.cuda.synchronize()
for _ in range(reps):
    sp.spmv_rows(d, x, y, 0, n)
torch.cuda.synchronize()
print("ok", float(y[12345]))
