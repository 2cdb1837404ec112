"""Files either side of the path: binary serialization and Matrix Market export
(stencil.hpp:61-64).  The C++ reader / writer (include/spmvcomp/io.hpp, host-only) against the numpy restatement
(oracle/serial.py): files of one are read by the other and written back byte for byte; file sizes follow the layout
formula; payload bytes per row are what `measured_cost` reports (K14)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1612_00530_b200")
TEST_IO = os.path.join(PKG, "test_io")
CLI = os.path.join(PKG, "spmvcomp_cli")
NAMES = ("stencil", "ell", "vt", "pattern", "pattern_values")


def oracle_files(orc, g):
    from oracle import serial
    m = orc.generate_matrix(*g)
    return m, {
        "stencil": serial.dump_stencil(m, g),
        "ell": serial.dump_ell(orc.to_ell(m)),
        "vt": serial.dump_vt(orc.compress_values(m)),
        "pattern": serial.dump_pattern(orc.compress_patterns(m, False)),
        "pattern_values": serial.dump_pattern(orc.compress_patterns(m, True)),
    }


@pytest.mark.parametrize("g", [(5, 4, 3), (1, 1, 1), (2, 2, 2), (7, 1, 4)])
def test_cpp_reader_and_writer_against_the_restatement(orc, g, tmp_path):
    from oracle import serial
    assert os.access(TEST_IO, os.X_OK), "test_io missing: run __graft_entry__.build()"
    m, files = oracle_files(orc, g)
    for k, b in files.items():
        (tmp_path / f"{k}.bin").write_bytes(b)
    r = subprocess.run([TEST_IO, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and ", 0 failed" in r.stdout, r.stdout + r.stderr
    for k, b in files.items():
        assert (tmp_path / f"{k}.bin.out").read_bytes() == b, k  # read and written back byte for byte
    assert (tmp_path / "matrix.mtx").read_text() == serial.matrix_market_text(m)
    # files the C++ side wrote from hand-built structures parse with the restatement
    f = serial.parse((tmp_path / "figure_vt.bin").read_bytes())
    assert f["sorted_columns"].tolist() == [45, 49, 51, 65, 50] and f["ends"].tolist() == [4, 5] and f["table"].tolist() == [-1.0, 26.0]
    f = serial.parse((tmp_path / "figure_pattern_rows.bin").read_bytes())
    assert f["patterns"][0][0].tolist() == [-5, -1, 1, 15, 0] and f["row_ends"].tolist() == [4, 5] and not f["values_in_pattern"]
    f = serial.parse((tmp_path / "one.bin").read_bytes())
    assert (f["n"], f["width"], f["nnz"], f["values"].tolist(), f["columns"].tolist()) == (1, 1, 1, [26.0], [0])


def test_file_sizes_follow_the_layout_and_the_byte_model(orc):
    """16-byte header, scalars, one 8-byte prefix per array; the payload per row is measured_cost's
    figure: ELL of 32^3 -> 324 exactly, vt -> 116, pattern -> 12 + o(1), pattern-values -> 4 + o(1)."""
    from oracle import serial
    g = (32, 32, 32)
    m, files = oracle_files(orc, g)
    n, nnz = m.n, m.nnz
    assert len(files["stencil"]) == 16 + 4 + (8 + 8 * (n + 1)) + (8 + 4 * nnz) + (8 + 8 * nnz) + 12
    assert len(files["ell"]) == 16 + 16 + 2 * 8 + 324 * n
    assert len(files["vt"]) == 16 + 8 + (8 + 16) + 2 * 8 + 116 * n
    dict_bytes = sum(8 + 4 * len(d) + 8 + 4 * len(e) for d, e in serial.parse(files["pattern_values"])["patterns"])
    assert len(files["pattern_values"]) == 16 + 4 + (8 + 16) + 8 + dict_bytes + (8 + 4 * n) + 1
    assert len(files["pattern"]) == len(files["pattern_values"]) + 8 + 8 * n
    for k, fmt in (("ell", orc.to_ell(m)), ("vt", orc.compress_values(m)), ("pattern", orc.compress_patterns(m, False)),
                   ("pattern_values", orc.compress_patterns(m, True))):
        assert serial.payload_bytes_per_row(files[k]) == pytest.approx(orc.measured_cost(fmt).bytes_per_row, rel=1e-12), k
    assert serial.payload_bytes_per_row(files["ell"]) == 324.0
    assert 4.0 < serial.payload_bytes_per_row(files["pattern_values"]) < 4.1
    assert 12.0 < serial.payload_bytes_per_row(files["pattern"]) < 12.1
    one = orc.generate_matrix(1, 1, 1)
    assert serial.payload_bytes_per_row(serial.dump_vt(orc.compress_values(one))) == 8.0


def test_restatement_round_trip(orc):
    from oracle import serial
    m, files = oracle_files(orc, (4, 3, 5))
    f = serial.parse(files["stencil"])
    assert f["n"] == m.n and np.array_equal(f["row_start"], m.row_start) and np.array_equal(f["cols"], m.cols)
    assert np.array_equal(f["vals"].view(np.uint64), m.vals.view(np.uint64)) and f["grid"] == (4, 3, 5)
    p = orc.compress_patterns(m, False)
    f = serial.parse(files["pattern"])
    assert np.array_equal(f["row_pattern"], p.row_pattern) and len(f["patterns"]) == p.n_patterns
    assert np.array_equal(f["row_ends"].reshape(m.n, p.m), p.ends_flat.reshape(p.n_patterns, p.m)[p.row_pattern])
    with pytest.raises(ValueError):
        serial.parse(b"NOTSPMVC" + files["ell"][8:])
    with pytest.raises(ValueError):
        serial.parse(files["ell"] + b"\0")


@pytest.mark.gpu
def test_cli_writes_and_reads_matrix_files(orc, tmp_path):
    """`generate --out` writes the device generator's matrix in the layout (bytes equal to the restatement's file of
    the oracle's matrix); `bench --matrix` / `solve --matrix` read it back and report what --grid reports."""
    import json
    from oracle import serial
    g = (24, 10, 12)
    path, mm = tmp_path / "m.bin", tmp_path / "m.mtx"
    r = subprocess.run([CLI, "generate", "--grid", *map(str, g), "--out", str(path), "--mm", str(mm)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    m = orc.generate_matrix(*g)
    assert path.read_bytes() == serial.dump_stencil(m, g)
    assert mm.read_text() == serial.matrix_market_text(m)
    assert json.loads(r.stdout)["file_bytes"] == path.stat().st_size
    outs = []
    for src in (["--grid", *map(str, g)], ["--matrix", str(path)]):
        r = subprocess.run([CLI, "bench", *src, "--format", "pattern-values", "--reps", "3"], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        outs.append(json.loads(r.stdout))
    assert outs[0]["checksum"] == outs[1]["checksum"] and outs[0]["grid"] == outs[1]["grid"] == list(g)
    assert outs[0]["compression_ratio"] == outs[1]["compression_ratio"]
    for fmt in ("ell", "vt", "pattern", "pattern-values"):  # bench --save writes the format's file as the restatement does
        fpath = tmp_path / f"{fmt}.bin"
        r = subprocess.run([CLI, "bench", "--matrix", str(path), "--format", fmt, "--reps", "1", "--save", str(fpath)], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        want = {"ell": lambda: serial.dump_ell(orc.to_ell(m)), "vt": lambda: serial.dump_vt(orc.compress_values(m)),
                "pattern": lambda: serial.dump_pattern(orc.compress_patterns(m, False)),
                "pattern-values": lambda: serial.dump_pattern(orc.compress_patterns(m, True))}[fmt]()
        assert fpath.read_bytes() == want, fmt
        assert json.loads(r.stdout)["file_bytes"] == len(want)
    r = subprocess.run([CLI, "solve", "--matrix", str(path), "--backend", "pattern"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and json.loads(r.stdout)["converged"] is True
    r = subprocess.run([CLI, "bench", "--matrix", str(tmp_path / "missing.bin"), "--format", "ell"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 1 and "cannot open" in r.stderr
