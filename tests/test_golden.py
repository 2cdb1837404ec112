"""Committed golden fixtures (tests/golden/spmv_golden.json, written by tests/golden/make_golden.py): the oracle must
reproduce them bit for bit on the CPU, and the device path must reproduce them bit for bit on the GPU."""
import hashlib
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "spmv_golden.json")) as f:
    GOLD = json.load(f)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hexes(a):
    return [format(int(v), "016x") for v in np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)]


def test_reference_known_answers_through_the_oracle(orc):
    k = GOLD["reference_known_answers"]["figure_row"]
    rows = [[(i, 26.0)] for i in range(66)]
    rows[k["row"]] = list(zip(k["columns"], k["values"]))
    m = orc.stencil_from_rows(66, rows)
    vt, pc = orc.compress_values(m), orc.compress_patterns(m)
    w = vt.width
    assert list(vt.table) == k["value_table"]
    assert list(vt.sorted_columns[k["row"] * w:k["row"] * w + 5]) == k["sorted_columns"]
    assert list(vt.ends[k["row"] * 2:k["row"] * 2 + 2]) == k["ends"]
    disp, _ = pc.pattern(int(pc.row_pattern[k["row"]]))
    assert list(disp) == k["displacements"]
    assert orc.spmv(pc, np.ones(66))[k["row"]] == k["y_for_ones"]
    bpr = GOLD["reference_known_answers"]["bytes_per_interior_row"]
    for name, fmt in (("ell", 0), ("vt", 1), ("pattern", 2), ("pattern-values", 3)):
        assert orc.format_cost(fmt, 27, 2).bytes_per_row == bpr[name]


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: "x".join(map(str, c["grid"])))
def test_oracle_reproduces_the_golden_streams_and_products(orc, case):
    g = tuple(case["grid"])
    m = orc.generate_matrix(*g)
    v = GOLD["vector"]
    x = orc.make_test_vector(m.n, orc.RANDOM, seed=v["seed"], lo=v["lo"], hi=v["hi"])
    assert (m.n, m.nnz) == (case["rows"], case["nnz"]) and hexes(x[:8]) == case["x_first8"] and sha(x) == case["x_sha256"]
    ell, vt, pc = orc.to_ell(m), orc.compress_values(m), orc.compress_patterns(m, True)
    assert (ell.width, sha(ell.values), sha(ell.columns)) == (case["ell"]["width"], case["ell"]["values_sha256"], case["ell"]["columns_sha256"])
    assert (hexes(vt.table), sha(vt.sorted_columns), sha(vt.ends)) == (case["vt"]["table"], case["vt"]["sorted_columns_sha256"], case["vt"]["ends_sha256"])
    p = case["pattern"]
    assert pc.n_patterns == p["n_patterns"] and [int(t) for t in pc.disp_offsets] == p["disp_offsets"]
    assert [int(t) for t in pc.disp_flat] == p["disp_flat"] and [int(t) for t in pc.ends_flat] == p["ends_flat"]
    assert sha(pc.row_pattern) == p["row_pattern_sha256"] and [int(t) for t in pc.row_pattern[:32]] == p["row_pattern_first32"]
    ys = {"ell": orc.spmv(ell, x), "vt": orc.spmv(vt, x), "pattern": orc.spmv(pc, x)}
    assert {k: sha(y) for k, y in ys.items()} == case["y_sha256"] and hexes(ys["pattern"][:8]) == case["y_pattern_first8"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: "x".join(map(str, c["grid"])))
def test_device_path_reproduces_the_golden_fixtures(case):
    """Generator, compressors, vector fill and the three SpMV kernels on the GPU against committed data only."""
    import paper_1612_00530_b200 as sp
    g = tuple(case["grid"])
    m = sp.generate_matrix(sp.GridSpec(*g))
    n = m.n
    v = GOLD["vector"]
    xd = sp.DeviceVector(n)
    sp.check(sp.lib.spmvb_vec_fill(sp.C.c_void_p(xd.ptr), n, sp.RANDOM, v["seed"], v["lo"], v["hi"], 0, None))
    x = xd.to_host()
    assert hexes(x[:8]) == case["x_first8"] and sha(x) == case["x_sha256"]
    ell, vt, pc = sp.to_ell(m), sp.compress_values(m), sp.compress_patterns(m, True)
    assert sha(ell.download("values")) == case["ell"]["values_sha256"] and sha(ell.download("columns")) == case["ell"]["columns_sha256"]
    assert sha(vt.download("sorted_columns")) == case["vt"]["sorted_columns_sha256"] and sha(vt.download("ends")) == case["vt"]["ends_sha256"]
    p = case["pattern"]
    assert [int(t) for t in pc.download("disp_flat")] == p["disp_flat"] and [int(t) for t in pc.download("ends_flat")] == p["ends_flat"]
    assert sha(pc.download("row_pattern")) == p["row_pattern_sha256"]
    for name, a in (("ell", ell), ("vt", vt), ("pattern", pc)):
        assert sha(sp.spmv(a, x)) == case["y_sha256"][name], name
    for march in (0, 90):  # the default dispatch and the tensor ring forced
        sp.set_option("box_march", march)
        try:
            assert sha(sp.spmv(pc, x)) == case["y_sha256"]["pattern"]
        finally:
            sp.set_option("box_march", 0)
