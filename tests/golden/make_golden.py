"""Generates tests/golden/spmv_golden.json from the CPU oracle (oracle/, itself pinned by the reference's worked
examples in tests/test_oracle_kat.py).  The fixture freezes, for a few small seeded cases, every stream of the three
formats and the SpMV results bit for bit, so that a change of the oracle or of the device path shows up as a diff
against committed data rather than only against each other.  Also recorded verbatim: the reference's own known
answers for the paper's figure row and the byte model.

    python tests/golden/make_golden.py      # rewrites the fixture; commit the result
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402

GRIDS = [(4, 4, 4), (6, 5, 7), (12, 10, 9), (70, 6, 9)]
SEED = 7


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hexes(a):
    return [format(int(v), "016x") for v in np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)]


def case(g):
    m = orc.generate_matrix(*g)
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=SEED, lo=-1.0, hi=1.0)
    ell, vt = orc.to_ell(m), orc.compress_values(m)
    pc = orc.compress_patterns(m, True)
    out = {
        "grid": list(g), "rows": int(m.n), "nnz": int(m.nnz), "x_first8": hexes(x[:8]), "x_sha256": sha(x),
        "ell": {"width": int(ell.width), "values_sha256": sha(ell.values), "columns_sha256": sha(ell.columns)},
        "vt": {"table": hexes(vt.table), "sorted_columns_sha256": sha(vt.sorted_columns), "ends_sha256": sha(vt.ends)},
        "pattern": {"n_patterns": int(pc.n_patterns), "table": hexes(pc.table), "disp_offsets": [int(v) for v in pc.disp_offsets],
                    "disp_flat": [int(v) for v in pc.disp_flat], "ends_flat": [int(v) for v in pc.ends_flat],
                    "row_pattern_sha256": sha(pc.row_pattern), "row_pattern_first32": [int(v) for v in pc.row_pattern[:32]]},
        "y_sha256": {"ell": sha(orc.spmv(ell, x)), "vt": sha(orc.spmv(vt, x)), "pattern": sha(orc.spmv(pc, x))},
        "y_pattern_first8": hexes(orc.spmv(pc, x)[:8]),
    }
    return out


def main():
    doc = {
        "generator": "tests/golden/make_golden.py (CPU oracle, gcc -O2 -ffp-contract=off)",
        "vector": {"kind": "random", "seed": SEED, "lo": -1.0, "hi": 1.0},
        "reference_known_answers": {  # stated by the reference itself, not computed here
            "figure_row": {"row": 50, "columns": [45, 49, 50, 51, 65], "values": [-1.0, -1.0, 26.0, -1.0, -1.0],
                           "value_table": [-1.0, 26.0], "sorted_columns": [45, 49, 51, 65, 50], "ends": [4, 5],
                           "displacements": [-5, -1, 1, 15, 0], "y_for_ones": 22.0},
            "bytes_per_interior_row": {"ell": 324, "vt": 116, "pattern": 12, "pattern-values": 4},
            "roofline_gflops_at_75_GBps": {"ell": 12.5, "vt": 34.9, "pattern": 337.5},
        },
        "cases": [case(g) for g in GRIDS],
    }
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "spmv_golden.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
