"""The command-line harness (SPEC.md:425-500 [MODULE] bench_cli): `spmvcomp_cli`.
model / generate / usage errors run anywhere; bench, solve and calibrate need the GPU."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1612_00530_b200", "spmvcomp_cli")


def run(*args):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout, r.stderr


def table(out):
    rows = {}
    for line in out.strip().splitlines()[1:]:
        f = line.split()
        rows[f[0]] = [float(v) for v in f[1:]]
    return rows


def test_cli_is_built():
    assert os.access(CLI, os.X_OK), "spmvcomp_cli missing: run __graft_entry__.build()"


def test_model_reproduces_the_paper_column():
    """`model --bandwidth 75` -> 12.5 / 34.9 / 337.5 (+ pattern-values) (K13)."""
    rc, out, _ = run("model", "--bandwidth", 75)
    assert rc == 0
    t = table(out)
    assert [t[k][0] for k in ("ell", "vt", "pattern", "pattern-values")] == [324.0, 116.0, 12.0, 4.0]
    assert t["ell"][2] == 12.5 and abs(t["vt"][2] - 34.9) < 0.05 and t["pattern"][2] == 337.5 and t["pattern-values"][2] == 1012.5
    rc, out2, _ = run("model", "--bandwidth", 150)
    t2 = table(out2)
    assert all(abs(t2[k][2] - 2 * t[k][2]) < 1e-3 * t[k][2] for k in t)  # linearity
    rc, out3, _ = run("model", "--bandwidth", 85, "--formats", "ell")
    assert abs(table(out3)["ell"][2] - 14.17) < 0.005


def test_generate_sizes_and_overflow_guard():
    rc, out, _ = run("generate", "--grid", 4, 4, 4)
    assert rc == 0 and json.loads(out)["rows"] == 64 and json.loads(out)["nnz"] == 1000
    rc, out, _ = run("generate", "--grid", 1, 1, 1)
    assert rc == 0 and json.loads(out) == {"grid": [1, 1, 1], "rows": 1, "nnz": 1, "csr_bytes": 28, "file_bytes": 0}
    rc, _, err = run("generate", "--grid", 100000, 100000, 100000)
    assert rc != 0 and "rows" in err  # SPEC.md:442 sizing error, nonzero exit


SCHEMA = os.path.join(ROOT, "paper_1612_00530_b200", "cpp", "report.schema.json")


def validate_report(text):
    """JSON reports validate against the schema shipped in the repo."""
    import jsonschema
    with open(SCHEMA) as f:
        schema = json.load(f)
    jsonschema.Draft202012Validator.check_schema(schema)
    obj = json.loads(text)
    jsonschema.validate(obj, schema)
    return obj


def test_generate_report_validates_against_the_schema():
    import jsonschema
    rc, out, _ = run("generate", "--grid", 4, 4, 4)
    assert rc == 0 and validate_report(out)["rows"] == 64
    with pytest.raises(jsonschema.ValidationError):
        validate_report('{"grid": [4, 4, 4], "rows": 64}')
    with pytest.raises(jsonschema.ValidationError):
        validate_report('{"backend": "csr", "preconditioner": "none", "grid": [4, 4, 4], "iterations": 1, "converged": true, '
                        '"final_residual": 0, "flops_total": 1}')


@pytest.mark.gpu
def test_reports_validate_and_land_in_the_report_directory(tmp_path):
    """bench / solve reports validate against the schema; the roofline column follows the configured bandwidth;
    SPMVCOMP_REPORT_DIR receives a copy of every report."""
    env = dict(os.environ, SPMVCOMP_REPORT_DIR=str(tmp_path))
    r = subprocess.run([CLI, "bench", "--grid", "32", "32", "32", "--format", "vt", "--reps", "3", "--bandwidth", "150"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr
    rep = validate_report(r.stdout)
    assert rep["machine_bandwidth_gbs"] == 150.0
    assert rep["roofline_gflops"] == pytest.approx(150.0 * (2 * rep["nnz"] / rep["rows"]) / rep["bytes_per_row"], rel=1e-5)
    assert (tmp_path / "bench_vt_32x32x32.json").read_text() == r.stdout
    rc, out, _ = run("bench", "--grid", 32, 32, 32, "--format", "pattern", "--reps", 2)
    assert validate_report(out)["machine_bandwidth_gbs"] == 75.0  # the reference's default MachineSpec (perf_model.hpp)
    r = subprocess.run([CLI, "bench", "--grid", "16", "16", "16", "--format", "ell", "--reps", "2", "--out", "csv"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and (tmp_path / "bench_ell_16x16x16.csv").read_text() == r.stdout
    assert r.stdout.splitlines()[0] == ("format,nx,ny,nz,repetitions,wall_time,achieved_gflops,effective_bandwidth_gbs,"
                                        "compression_ratio,bytes_per_row,checksum")
    r = subprocess.run([CLI, "solve", "--grid", "16", "16", "16", "--backend", "vt"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and validate_report(r.stdout)["converged"] is True
    assert (tmp_path / "solve_vt_16x16x16.json").read_text() == r.stdout
    plain = validate_report(r.stdout)
    rc, out, err = run("solve", "--grid", 16, 16, 16, "--backend", "vt", "--precond", "symgs")  # SPEC.md:456 precond
    pre = validate_report(out)
    assert rc == 0 and pre["converged"] and pre["preconditioner"] == "symgs" and pre["iterations"] < plain["iterations"]
    rc, out, _ = run("solve", "--grid", 16, 16, 16, "--precond", "symgs:2")
    assert rc == 0 and validate_report(out)["iterations"] <= pre["iterations"]
    rc, _, err = run("solve", "--grid", 16, 16, 16, "--precond", "jacobi")
    assert rc == 2 and err
    env["SPMVCOMP_REPORT_DIR"] = str(tmp_path / "missing")
    r = subprocess.run([CLI, "solve", "--grid", "8", "8", "8"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 1 and "cannot write the report" in r.stderr


def test_usage_errors_exit_2():
    for args in (("frobnicate",), (), ("bench", "--grid", 4, 4), ("model",), ("bench", "--grid", 4, 4, 4, "--format", "csr5"),
                 ("bench", "--format", "ell"), ("bench", "--grid", 4, 4, 4, "--matrix", "m.bin", "--format", "ell"),
                 ("solve", "--grid", 4, 4, 4, "--max-iter", 0)):
        rc, _, err = run(*args)
        assert rc == 2 and err, args


@pytest.mark.gpu
def test_bench_reports_and_compression_ratios():
    reps = {}
    for fmt in ("ell", "vt", "pattern", "pattern-values"):
        rc, out, err = run("bench", "--grid", 32, 32, 32, "--format", fmt, "--reps", 10)
        assert rc == 0, err
        reps[fmt] = json.loads(out)
        assert reps[fmt]["achieved_gflops"] > 0 and reps[fmt]["repetitions"] == 10
        assert reps[fmt]["max_scaled_deviation_vs_ell"] <= 1e-12
    assert abs(reps["vt"]["compression_ratio"] - 324 / 116) <= 0.02 * 324 / 116
    assert abs(reps["pattern-values"]["compression_ratio"] - 81) <= 0.05 * 81
    assert reps["pattern"]["compression_ratio"] == 27.0 and reps["ell"]["compression_ratio"] == 1.0
    rc, out1, _ = run("bench", "--grid", 32, 32, 32, "--format", "vt", "--reps", 1)
    assert json.loads(out1)["checksum"] == reps["vt"]["checksum"]                      # SPEC.md:452 determinism
    rc, csv, _ = run("bench", "--grid", 16, 16, 16, "--format", "pattern", "--reps", 2, "--out", "csv")
    head, row = csv.strip().splitlines()
    assert rc == 0 and head.split(",")[:5] == ["format", "nx", "ny", "nz", "repetitions"] and row.startswith("pattern,16,16,16,2,")


@pytest.mark.gpu
def test_solve_backend_invariance_and_exit_codes():
    its = {}
    for backend in ("ell", "vt", "pattern"):
        rc, out, err = run("solve", "--grid", 16, 16, 16, "--backend", backend, "--tol", 1e-8)
        assert rc == 0, err
        rep = json.loads(out)
        assert rep["converged"] is True and rep["final_residual"] <= 1e-8
        its[backend] = rep["iterations"]
    assert its["ell"] == its["pattern"] == its["vt"]
    rc, out, _ = run("solve", "--grid", 16, 16, 16, "--max-iter", 1)
    assert rc == 1 and json.loads(out)["converged"] is False


@pytest.mark.gpu
def test_calibrate_reports_a_positive_stable_bandwidth():
    a = json.loads(run("calibrate")[1])["device_stream_bandwidth_gbs"]
    b = json.loads(run("calibrate")[1])["device_stream_bandwidth_gbs"]
    assert a > 0 and abs(a - b) <= 0.2 * max(a, b)


def test_model_table_csv_and_json():
    """model_table / model_table_csv / model_table_json (inc/perf_model.hpp:82-95): fixed CSV column order."""
    rc, out, _ = run("model", "--bandwidth", 75, "--out", "csv")
    assert rc == 0
    lines = out.strip().splitlines()
    assert lines[0] == "format,bytes_per_row,bytes_per_flop,predicted_gflops,limiting_resource"
    rows = {ln.split(",")[0]: ln.split(",") for ln in lines[1:]}
    assert list(rows) == ["ell", "vt", "pattern", "pattern-values"]
    assert float(rows["ell"][1]) == 324.0 and float(rows["ell"][3]) == 12.5 and rows["ell"][4] == "bandwidth"
    assert float(rows["pattern"][3]) == 337.5 and float(rows["pattern-values"][1]) == 4.0
    rc, out, _ = run("model", "--bandwidth", 75, "--out", "json", "--formats", "vt,ell")
    assert rc == 0
    t = json.loads(out)
    assert [r["format"] for r in t] == ["vt", "ell"] and t[0]["bytes_per_row"] == 116.0 and abs(t[0]["predicted_gflops"] - 34.9) < 0.05
    assert t[1]["flops_per_row"] == 54.0 and t[1]["limiting_resource"] == "bandwidth"


def test_machine_spec_file_round_trips_into_model(tmp_path):
    """The machine-spec file read back by `model --machine`: same table as --bandwidth."""
    spec = tmp_path / "spec.json"
    spec.write_text('{"read_bandwidth": 75000000000}\n')
    rc, out, _ = run("model", "--machine", str(spec))
    rc2, out2, _ = run("model", "--bandwidth", 75)
    assert rc == 0 and rc2 == 0 and out == out2
    bad = tmp_path / "bad.json"
    bad.write_text('{"peak_flops": 1e12}\n')
    rc, _, err = run("model", "--machine", str(bad))
    assert rc == 1 and "read_bandwidth" in err
    rc, _, err = run("model", "--machine", str(tmp_path / "missing.json"))
    assert rc == 1


@pytest.mark.gpu
def test_calibrate_writes_a_machine_spec_that_bench_reads(tmp_path):
    spec = tmp_path / "spec.json"
    rc, out, err = run("calibrate", "--out", str(spec))
    assert rc == 0, err
    gbs = json.loads(out)["device_stream_bandwidth_gbs"]
    assert gbs > 0
    saved = json.loads(spec.read_text())
    assert abs(saved["read_bandwidth"] / 1e9 - gbs) < 1e-3 * gbs
    rc2, out2, _ = run("calibrate")
    assert rc2 == 0 and abs(json.loads(out2)["device_stream_bandwidth_gbs"] - gbs) < 0.2 * gbs  # two runs within 20 %
    rc, out, err = run("bench", "--grid", 32, 32, 32, "--format", "pattern-values", "--reps", 5, "--machine", str(spec))
    assert rc == 0, err
    rep = json.loads(out)
    assert abs(rep["machine_bandwidth_gbs"] - saved["read_bandwidth"] / 1e9) < 1e-6 * rep["machine_bandwidth_gbs"]
    assert abs(rep["roofline_gflops"] - rep["machine_bandwidth_gbs"] * (2.0 * rep["nnz"] / rep["rows"]) / rep["bytes_per_row"]) < 1e-3 * rep["roofline_gflops"]
