#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200-native compressed SpMV path.

Workload (BASELINE.json configs[2]): HPCG 27-point stencil, 256x256x256 rows per
GPU stacked as z-slabs (global nz = 256*G), compressed pattern format (4-byte
pattern id per row + dictionary), x ~ U[-1,1) from seed 7, fp64.  One "step" is
one SpMV y = A x over the slab (plus the one-plane halo exchange when G > 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

`--gpus N` with N > 1 and no torchrun environment starts the N ranks itself (re-exec
under torch.distributed.run on 127.0.0.1).  Prints ONE JSON line (rank 0).  At N = 1
the line also carries `configs`: one block per BASELINE config that fits one GPU
(C1 32^3 ELL, C2 128^3 all formats, C4 perturbed 128^3 hybrid, C5 512^3 pattern), each
with its own parity result against the CPU oracle, kernel time, algorithmic bytes,
roofline fraction and regime (L2-resident or HBM).  `--impl reference` times the CPU
restatement of the reference's unchecked::spmv_rows (the oracle; the reference ships
no src/) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 7
METRIC = "SpMV GFLOP/s (2*nnz/t), fp64, HPCG 27-point stencil, compressed pattern format"
PERTURB = (11, 0.1, 0.1)  # BASELINE configs[3]: seed, fraction of rows, noise


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--grid", type=int, nargs=3, default=[256, 256, 256], help="rows per GPU (nx ny nz_local)")
    ap.add_argument("--exchange", default=os.environ.get("SPMVB_EXCHANGE", "p2p"), choices=["nccl", "p2p"],
                    help="N > 1: halo planes pulled from CUDA-IPC-mapped neighbour memory over NVLink (falls back to nccl when "
                         "a rank cannot map its neighbours), or NCCL send/recv")
    ap.add_argument("--schedule", default=os.environ.get("SPMVB_SCHEDULE", "serial"), choices=["serial", "overlap"],
                    help="N > 1: exchange then one launch, or exchange || interior planes then the two boundary planes")
    ap.add_argument("--no-graph", action="store_true", help="N > 1, nccl: do not capture the step into a CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-formats", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config blocks (C1, C2, C4, C5)")
    return ap.parse_args()


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs, copy kernel)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(grid, kernel_family):
    """dram bytes per launch of the dominant kernel from the committed ncu capture -- only when that capture was taken
    on this grid and kernel (profiles/latest_traffic.json names both); null otherwise."""
    path = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            t = json.load(f)
        if list(t.get("grid", [256, 256, 256])) == list(grid) and t.get("kernel_family", 9) == kernel_family:
            return t.get("dram_bytes_per_launch")
    return None


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons through NVML while the GPU runs the timed loops."""

    def __init__(self, index):
        super().__init__(daemon=True)
        self.index, self.stop_flag, self.samples, self.reasons, self.max_mhz = index, False, [], set(), None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def run(self):
        if self.nv is None:
            return
        nv = self.nv
        names = {}
        for attr, name in (("HwSlowdown", "hw_slowdown"), ("HwThermalSlowdown", "hw_thermal_slowdown"),
                           ("SwThermalSlowdown", "sw_thermal_slowdown"), ("SwPowerCap", "sw_power_cap"),
                           ("HwPowerBrakeSlowdown", "hw_power_brake")):
            bit = getattr(nv, "nvmlClocksEventReason" + attr, None) or getattr(nv, "nvmlClocksThrottleReason" + attr, None)
            if bit is not None:
                names[bit] = name
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons", None)
        while not self.stop_flag:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = get_reasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.0005)

    def result(self):
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def nnz_slab(nx, ny, nz_global, z0, z1):
    """Exact nonzero count of planes [z0,z1) of the global stencil."""
    per_plane = lambda k: (3 * nx - 2) * (3 * ny - 2) * k  # noqa: E731
    total = 0
    for z in range(z0, z1):
        total += per_plane(min(z + 1, nz_global - 1) - max(z - 1, 0) + 1)
    return total


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal"):
                    ram = round(int(ln.split()[1]) / 2 ** 20, 1)
                    break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "ram_gib": ram}


def workload_name(nx, ny, nz, g):
    return (f"BASELINE configs[2]: HPCG 27-point stencil {nx}x{ny}x{nz} per GPU, {g} z-slab(s) "
            f"(global {nx}x{ny}x{nz * g}), diagonal 26 / off-diagonal -1, x~U[-1,1) seed {SEED}")


def l2_cache_bytes():
    """cudaDevAttrL2CacheSize of device 0 (both arms run on the GPU box); None without a device."""
    try:
        import torch
        if torch.cuda.is_available():
            return int(torch.cuda.get_device_properties(0).L2_cache_size)
    except Exception:  # noqa: BLE001
        pass
    return None


def l2_note(alg_bytes, l2_bytes):
    if l2_bytes is None:
        return f"inputs: {alg_bytes / 1e6:.0f} MB per SpMV (no CUDA device visible: L2 size unknown)"
    if alg_bytes <= 0.8 * l2_bytes:
        return (f"inputs ({alg_bytes / 1e6:.0f} MB per SpMV) fit the {l2_bytes / 1e6:.0f} MB L2 (cudaDevAttrL2CacheSize): repeated SpMVs are "
                "L2-resident and no flush is made -- the HBM fraction is not the binding limit for this grid")
    return (f"inputs ({alg_bytes / 1e6:.0f} MB per SpMV: 20 B/row) exceed the {l2_bytes / 1e6:.0f} MB L2 (cudaDevAttrL2CacheSize); "
            "no flush needed between steps")


def make_config(nx, ny, nz, g):
    """The `config` object, identical in both arms (the driver compares them)."""
    return {"workload": workload_name(nx, ny, nz, g),
            "format": "pattern (values_in_pattern): 4-byte pattern id per row + 27-entry dictionary",
            "rows_per_gpu": nx * ny * nz, "n_gpus": g, "l2": l2_note(20.0 * nx * ny * nz, l2_cache_bytes())}


# ------------------------------------------------------------------------------------------------
def cpu_sample(nx, ny, nz, steps, warmup, budget_s, threads=None, pc=None, x=None):
    """Times the oracle's pattern SpMV (CPU restatement of unchecked::spmv_rows, kernels.hpp:35-36) with `threads` host
    threads (default: all) on a bounded sample of the workload: the centre planes that `budget_s` seconds allow."""
    import numpy as np
    from oracle import oracle as orc

    cores = threads or os.cpu_count() or 1
    if pc is None:
        pc = orc.compress_patterns_grid(nx, ny, nz, values_in_pattern=True)
        x = orc.make_test_vector(pc.n, orc.RANDOM, seed=SEED, lo=-1.0, hi=1.0)
    n = pc.n
    y = np.zeros(n)
    plane = nx * ny
    t0 = time.perf_counter()
    orc.spmv_rows(pc, x, y, 0, n, threads=cores)  # warm-up pass, also sizes the sample
    t_full = time.perf_counter() - t0
    frac = min(1.0, budget_s / max(t_full * (steps + warmup), 1e-9))
    planes = max(2, min(nz, int(nz * frac)))
    z0 = (nz - planes) // 2  # interior planes: 27 nnz rows dominate as in the full workload
    b, e = z0 * plane, (z0 + planes) * plane
    nnz = nnz_slab(nx, ny, nz, z0, z0 + planes)
    for _ in range(warmup):
        orc.spmv_rows(pc, x, y, b, e, threads=cores)
    # The host cores of a GPU box are virtual and noisy: the same loop has read 23 and 49 GFLOP/s minutes apart on one box, slow for
    # seconds at a time.  The loop of `steps` passes is therefore repeated for up to ~12 s (at most 20 times) and the fastest loop is
    # reported: noise can only slow the CPU arm down, and the faster reading is the one a GPU / CPU ratio should be held against.
    loops, dt = [], None
    t_begin = time.perf_counter()
    while len(loops) < 20:
        t0 = time.perf_counter()
        for _ in range(steps):
            orc.spmv_rows(pc, x, y, b, e, threads=cores)
        loops.append(time.perf_counter() - t0)
        if time.perf_counter() - t_begin + loops[-1] > min(12.0, 2.0 * budget_s):
            break
    dt = min(loops)
    per_pass = sorted(t / steps * 1e3 for t in loops)
    return {"gflops": 2.0 * nnz * steps / dt / 1e9, "ms_per_step": dt / steps * 1e3, "cores": cores,
            "gbs": 20.0 * (e - b) * steps / dt / 1e9,
            "sample": f"pattern-format SpMV over planes [{z0},{z0 + planes}) of {nx}x{ny}x{nz} "
                      f"({e - b} rows, {nnz} nnz) x {steps} reps after {warmup + 1} warm-up passes, {cores} threads (contiguous row ranges); "
                      f"fastest of {len(loops)} such loops (ms per pass: min {per_pass[0]:.1f}, median {per_pass[len(per_pass) // 2]:.1f}, max {per_pass[-1]:.1f})",
            "pc": pc, "x": x}


def cpu_baseline_block(nx, ny, nz, steps=20, warmup=3, budget_s=20.0):
    """cpu_baseline for the JSON line: all host threads (the value) and one thread, CPU model and RAM."""
    r = cpu_sample(nx, ny, nz, steps, warmup, budget_s)
    r1 = cpu_sample(nx, ny, nz, max(2, steps // 6), 1, budget_s / 2, threads=1, pc=r["pc"], x=r["x"])
    block = {"value": r["gflops"], "unit": "GFLOP/s", "cores": r["cores"], "kind": "port", "sample": r["sample"],
             "algorithmic_gbs": r["gbs"], "ms_per_step": r["ms_per_step"],
             "single_thread": {"value": r1["gflops"], "unit": "GFLOP/s", "cores": 1, "ms_per_step": r1["ms_per_step"],
                               "sample": r1["sample"]},
             "host": host_info()}
    return block, r


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nx, ny, nz = args.grid
    # bounded: the centre planes that fit ~150 s for steps + warmup passes (the whole grid at the driver's settings)
    block, r = cpu_baseline_block(nx, ny, nz, steps=args.steps, warmup=args.warmup, budget_s=150.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": r["gflops"], "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": make_config(nx, ny, nz, args.gpus),
        "note": "CPU restatement of the reference's unchecked::spmv_rows (the reference ships no implementation source); "
                "host threads only, no GPU",
        "cpu_baseline": block,
        "e2e": {"value": r["gflops"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
KERNEL_NAMES = {1: "spmv_pattern_generic_kernel (List 1 as written)", 2: "spmv_pattern_box_kernel (one-column sliding window)",
                3: "spmv_pattern_box3_kernel (register sliding window)", 4: "lab variant",
                9: "spmv_pattern_ringp_kernel (persistent TMA tensor ring)"}


def time_loop(torch, stream, fn, reps, warm=3):
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    stream.synchronize()
    return e0.elapsed_time(e1) / reps


def time_graph(torch, stream, fn, reps):
    """The same loop recorded once into a CUDA graph and replayed: per-launch host overhead leaves the measurement
    (graph-launched rep loop for the configurations whose kernels take a few microseconds)."""
    fn()
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps):
            fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):  # replay() launches on the current stream: both replays on `stream`, never side by side
        g.replay()
        stream.synchronize()
        e0.record(stream)
        g.replay()
        e1.record(stream)
    stream.synchronize()
    return e0.elapsed_time(e1) / reps


def config_blocks(sp, torch, stream, peak, l2_bytes):
    """One block per BASELINE config that fits one GPU besides the headline: its own build, parity against the CPU
    oracle on the same seeded inputs (bit-exact: ids / index streams and y), kernel time, algorithmic bytes, frac."""
    import numpy as np
    from oracle import oracle as orc

    cores = os.cpu_count() or 1
    out = []

    def bits(a):
        return np.ascontiguousarray(a).view(np.uint64)

    def measure(a, x, y, n, reps, x_col0=0, x_len=None):
        fn = lambda: sp.spmv_rows(a, x, y, 0, n, x_col0=x_col0, x_len=n if x_len is None else x_len, stream=stream)  # noqa: E731
        direct = time_loop(torch, stream, fn, reps)
        try:
            graph = time_graph(torch, stream, fn, reps)
        except Exception:  # noqa: BLE001
            graph = None
        return direct, graph

    def block(name, fmt, grid, n, nnz, alg_bytes, ms_direct, ms_graph, parity, reps, extra=None):
        ms = min(ms_direct, ms_graph) if ms_graph else ms_direct
        fits = alg_bytes <= 0.8 * l2_bytes
        b = {"config": name, "format": fmt, "grid": list(grid), "rows": n, "nnz": nnz, "reps": reps,
             "kernel_ms": ms, "kernel_ms_direct_launches": ms_direct, "kernel_ms_graph_replay": ms_graph,
             "gflops": 2.0 * nnz / ms / 1e6, "algorithmic_bytes": alg_bytes, "algorithmic_gbs": alg_bytes / ms / 1e6,
             "frac_of_hbm_peak": alg_bytes / ms / 1e6 / peak,
             "regime": (f"L2-resident: {alg_bytes / 1e6:.1f} MB per SpMV fit the {l2_bytes / 1e6:.0f} MB L2 over the repetitions, so the HBM "
                        "fraction is not the binding limit (launch latency / L2 bandwidth is)") if fits else
                       f"HBM: {alg_bytes / 1e6:.1f} MB per SpMV exceed the {l2_bytes / 1e6:.0f} MB L2",
             "parity": parity}
        if extra:
            b.update(extra)
        out.append(b)

    # ---- C1: 32^3, uncompressed ELL, 1 GPU vs the CPU reference
    g = (32, 32, 32)
    m = orc.generate_matrix(*g)
    n = m.n
    xh = orc.make_test_vector(n, orc.RANDOM, seed=SEED, lo=-1.0, hi=1.0)
    ell_o = orc.to_ell(m)
    dm = sp.generate_matrix(sp.GridSpec(*g), stream=stream)
    ell = sp.to_ell(dm, stream=stream)
    x, y = sp.DeviceVector.from_host(xh), sp.DeviceVector(n)
    sp.spmv_rows(ell, x, y, 0, n, stream=stream)
    stream.synchronize()
    par = {"values_stream_identical": ell.download("values").tobytes() == ell_o.values.tobytes(),
           "columns_stream_identical": ell.download("columns").tobytes() == ell_o.columns.tobytes(),
           "rows_differing_from_cpu_oracle": int((bits(y.to_host()) != bits(orc.spmv(ell_o, xh))).sum())}
    d, gr = measure(ell, x, y, n, 100)
    yo = np.zeros(n)
    t0 = time.perf_counter()
    for _ in range(100):
        orc.spmv_rows(ell_o, xh, yo, 0, n, threads=cores)
    cpu_ms = (time.perf_counter() - t0) / 100 * 1e3
    block("C1 (BASELINE configs[0])", "ELL (fp64 values + int32 columns, width 27)", g, n, m.nnz, 340.0 * n, d, gr, par, 100,
          {"cpu_oracle_ms": cpu_ms, "cpu_oracle_gflops": 2.0 * m.nnz / cpu_ms / 1e6, "cpu_threads": cores})
    del ell, dm, x, y

    # ---- C2: 128^3, pattern / vt / ELL, 100 repetitions
    g = (128, 128, 128)
    m = orc.generate_matrix(*g)
    n = m.n
    xh = orc.make_test_vector(n, orc.RANDOM, seed=SEED, lo=-1.0, hi=1.0)
    dm = sp.generate_matrix(sp.GridSpec(*g), stream=stream)
    x, y = sp.DeviceVector.from_host(xh), sp.DeviceVector(n)
    for fmt, name, dev, ref, streams, bpr in (
            ("pattern", "pattern (values_in_pattern): ids + dictionary", sp.compress_patterns(dm, True, stream=stream),
             orc.compress_patterns(m, True), ("row_pattern", "disp_flat", "ends_flat"), 20.0),
            ("vt", "value table: sorted columns + group ends", sp.compress_values(dm, stream=stream), orc.compress_values(m),
             ("sorted_columns", "ends"), 132.0),
            ("ell", "ELL (fp64 values + int32 columns, width 27)", sp.to_ell(dm, stream=stream), orc.to_ell(m), ("values", "columns"), 340.0)):
        sp.spmv_rows(dev, x, y, 0, n, stream=stream)
        stream.synchronize()
        par = {f"{s}_stream_identical": dev.download(s).tobytes() == getattr(ref, s).tobytes() for s in streams}
        par["rows_differing_from_cpu_oracle"] = int((bits(y.to_host()) != bits(orc.spmv(ref, xh, threads=cores))).sum())
        d, gr = measure(dev, x, y, n, 100)
        extra = {"kernel": KERNEL_NAMES.get(sp.get_option("last_pattern_kernel"))} if fmt == "pattern" else None
        block("C2 (BASELINE configs[1])", name, g, n, m.nnz, bpr * n, d, gr, par, 100, extra)
        del dev, ref
    t_ell = out[-1]["kernel_ms"]
    for b in out[-3:]:
        b["speedup_over_uncompressed_ell"] = t_ell / b["kernel_ms"]
    del dm, m

    # ---- C4: 128^3 with 10 % of the rows perturbed: hybrid format (dictionary rows + uncompressed exception rows)
    mo = orc.generate_matrix(*g, perturb=PERTURB)
    ho = orc.compress_patterns(mo, True, min_pattern_rows=2)
    dm = sp.generate_matrix(sp.GridSpec(*g), perturb=PERTURB, stream=stream)
    hyb = sp.compress_patterns(dm, True, min_pattern_rows=2, stream=stream)
    info = hyb.info
    sp.spmv_rows(hyb, x, y, 0, n, stream=stream)
    stream.synchronize()
    par = {f"{s}_stream_identical": hyb.download(s).tobytes() == getattr(ho, s).tobytes()
           for s in ("row_pattern", "exc_rows", "exc_values", "exc_columns")}
    par["rows_differing_from_cpu_oracle"] = int((bits(y.to_host()) != bits(orc.spmv(ho, xh, threads=cores))).sum())
    alg = 20.0 * n + info.n_exc * (4.0 + 12.0 * info.w_exc)
    d, gr = measure(hyb, x, y, n, 100)
    ell4 = sp.to_ell(dm, stream=stream)
    d4, g4 = measure(ell4, x, y, n, 50)
    w4 = ell4.info.width
    block("C4 (BASELINE configs[3])", "hybrid: pattern ids + dictionary, exception rows as an ELL block", g, n, mo.nnz, alg, d, gr, par, 100,
          {"exception_rows": info.n_exc, "exception_width": info.w_exc, "dictionary_patterns": info.n_patterns,
           "uncompressed_ell_width": w4, "uncompressed_ell_ms": min(d4, g4) if g4 else d4,
           "speedup_over_uncompressed_ell": (min(d4, g4) if g4 else d4) / (min(d, gr) if gr else d),
           "note": "exception rows, the selection rule and the perturbation recipe are extensions (parity unpinned by the reference; DESIGN.md 4-5)"})
    del hyb, ell4, dm, mo, ho, x, y

    # ---- C5 at one GPU: 512^3, pattern format, 50 repetitions (x + y + ids = 2.7 GB; the CSR and ELL are never built)
    g = (512, 512, 512)
    n = g[0] * g[1] * g[2]
    plane = g[0] * g[1]
    nnz = nnz_slab(g[0], g[1], g[2], 0, g[2])
    big = sp.MultiSlab(sp.GridSpec(*g), [0])  # device-side build in one piece: generator -> compressor, CSR freed
    _, _, _, a, xg, yg = big.part(0)
    big.fill_x(sp.RANDOM, SEED, -1.0, 1.0)
    fn = lambda: sp.spmv_rows(a, xg, yg, 0, n, x_col0=-plane, x_len=n + 2 * plane, stream=stream)  # noqa: E731
    fn()
    stream.synchronize()
    # chunked parity at full size: the oracle regenerates and compresses chunks of 8 planes (2.1 M rows) of the
    # global grid -- first, last, and two inside -- ids compared through the dictionaries, y bit for bit
    yd = big.download_y()
    ids = a.download("row_pattern")
    off, flat = a.download("disp_offsets"), a.download("disp_flat")
    shapes = [tuple(flat[off[q]:off[q + 1]].tolist()) for q in range(a.info.n_patterns)]
    bad_y = bad_id = rows_checked = 0
    for z0 in (0, 200, 389, g[2] - 8):
        r0, r1 = z0 * plane, (z0 + 8) * plane
        co = orc.compress_patterns(orc.generate_matrix(*g, row_begin=r0, row_end=r1), True, row_offset=r0)
        oshapes = [tuple(co.disp_flat[co.disp_offsets[q]:co.disp_offsets[q + 1]].tolist()) for q in range(len(co.disp_offsets) - 1)]
        to_dev = np.array([shapes.index(s) for s in oshapes], dtype=np.int32)  # chunk numbering -> whole-matrix numbering
        bad_id += int((to_dev[co.row_pattern] != ids[r0:r1]).sum())
        lo, hi = max(r0 - plane, 0), min(r1 + plane, n)
        xl = orc.make_test_vector(hi - lo, orc.RANDOM, seed=SEED, lo=-1.0, hi=1.0, first_index=lo)
        yo = np.zeros(r1 - r0)
        orc.spmv_rows(co, xl, yo, 0, r1 - r0, x_col0=lo, threads=cores)
        bad_y += int((bits(yo) != bits(yd[r0:r1])).sum())
        rows_checked += r1 - r0
    par = {"rows_checked_against_cpu_oracle": rows_checked, "rows_differing_from_cpu_oracle": bad_y,
           "pattern_ids_differing_from_cpu_oracle": bad_id, "dictionary_patterns": a.info.n_patterns,
           "how": "4 chunks of 8 planes regenerated and compressed by the oracle; ids mapped through the dictionaries"}
    d = time_loop(torch, stream, fn, 50)
    kern = KERNEL_NAMES.get(sp.get_option("last_pattern_kernel"))
    block("C5 at 1 GPU (BASELINE configs[4])", "pattern (values_in_pattern): ids + dictionary", g, n, nnz, 20.0 * n, d, None, par, 50,
          {"kernel": kern})
    del big
    return out


# ------------------------------------------------------------------------------------------------
def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device; the B200 path has no CPU fallback")
    if world > 1 and torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} CUDA device(s) on this node")
    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import paper_1612_00530_b200 as sp
    sp.check(sp.lib.spmvb_set_device(local_rank))

    nx, ny, nzl = args.grid
    L = sp.SlabLayout(nx, ny, nzl * world, rank, world)
    n, plane = L.n_local, L.plane
    z0, z1 = L.z_range
    nnz_local = nnz_slab(nx, ny, nzl * world, z0, z1)
    main = torch.cuda.Stream()
    comm = torch.cuda.Stream()
    K, W = args.steps, max(args.warmup, 3)
    l2_bytes = torch.cuda.get_device_properties(local_rank).L2_cache_size

    with torch.cuda.stream(main):
        # ---- build on the device: generator -> compressor (+ dictionary merge across slabs)
        t_build = time.perf_counter()
        pc, csr = sp.build_slab_pattern(sp, L, dist if world > 1 else None, keep_csr=True, stream=main)
        assert pc.info.nnz == nnz_local, (pc.info.nnz, nnz_local)
        ell = sp.to_ell(csr, min_width=27, stream=main)
        xv = sp.DeviceVector(L.x_len)  # cudaMalloc'ed: can be mapped by the neighbours (--exchange p2p)
        x = torch.as_tensor(xv, device="cuda")  # zero-copy view: NCCL sends / receives slices of it
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        y2 = torch.empty(n, dtype=torch.float64, device="cuda")
        scale = torch.empty(n, dtype=torch.float64, device="cuda")
        sp.check(sp.lib.spmvb_vec_fill(x.data_ptr(), L.x_len, sp.RANDOM, SEED, -1.0, 1.0, L.x_col0, main.cuda_stream))
        main.synchronize()
        build_s = time.perf_counter() - t_build

        def kernel_of(a):
            def k(xl, yl, b, e):
                sp.spmv_rows(a, xl, yl, b, e, x_col0=L.x_col0, x_len=L.x_len, stream=main)
            return k

        slab = sp.DeviceSlabSpmv(sp, L, pc, dist if world > 1 else None, main, comm, torch, exchange=args.exchange,
                                 schedule=args.schedule)
        if world > 1 and args.exchange == "p2p":  # all ranks map their neighbours, or all fall back to NCCL send/recv
            try:
                slab.map_neighbours(x)
                mapped = 1
            except Exception as ex:  # noqa: BLE001
                print(f"rank {rank}: cannot map the neighbours' vectors ({ex}); falling back to --exchange nccl", file=sys.stderr)
                mapped = 0
            ok = torch.tensor([mapped], device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if not int(ok.item()):
                slab.unmap_neighbours()
                args.exchange = "nccl"
                slab = sp.DeviceSlabSpmv(sp, L, pc, dist, main, comm, torch, exchange="nccl", schedule=args.schedule)
            main.synchronize()
            dist.barrier()  # every rank's x is filled before anyone pulls a plane of it
        whole = kernel_of(pc)
        step = (lambda: whole(x, y, 0, n)) if world == 1 else (lambda: slab.spmv(x, y))

        # ---- verification gate: no number for a kernel that failed parity
        step()
        sp.spmv_rows(ell, x, y2, 0, n, x_col0=L.x_col0, x_len=L.x_len, stream=main)
        sp.row_abs_scale(csr, x, scale, x_col0=L.x_col0, stream=main)
        worst_vs_ell, _ = sp.compare(y, y2, n, scale=scale, stream=main)
        sp.set_option("pattern_kernel", 1)  # the plain List-1 kernel must agree bit for bit
        sp.spmv_rows(pc, x, y2, 0, n, x_col0=L.x_col0, x_len=L.x_len, stream=main)
        sp.set_option("pattern_kernel", 0)
        _, bits_vs_generic = sp.compare(y, y2, n, stream=main)
        if not (worst_vs_ell <= 1e-12) or bits_vs_generic != 0:
            raise sp.VerificationError(f"rank {rank}: compressed SpMV failed parity: max scaled deviation vs ELL "
                                       f"{worst_vs_ell:.3e}, {bits_vs_generic} rows differ from the List-1 kernel")
        del csr, scale

        # ---- timed region: K steps, device events, max over ranks
        sampler = ClockSampler(local_rank)  # started before the warm-up so that its thread set-up is not in the timed region
        sampler.start()
        for _ in range(W):
            step()
        graphed = False
        if world > 1 and args.exchange == "nccl" and not args.no_graph:
            main.synchronize()
            graphed = slab.capture(x, y)  # the whole step (send/recv + launches) as one graph launch per SpMV
            ok = torch.tensor([int(graphed)], device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # all ranks or none
            if not int(ok.item()):
                slab._graph, graphed = None, False
            for _ in range(2):
                step()
        main.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler.samples.clear()  # keep only what is sampled from here on: the timed region and the kernel-alone loops
        sampler.reasons.clear()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(main)
        for _ in range(K):
            step()
        ev1.record(main)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        launches = K * slab.launches_per_spmv
        family = sp.get_option("last_pattern_kernel")

        # ---- dominant kernel alone (roofline): all local rows, no exchange
        kernel_ms = time_loop(torch, main, lambda: whole(x, y, 0, n), max(K, 50))

        # ---- other formats, same x (context for the compression gain)
        extra = {}
        if not args.no_extra_formats:
            def time_fmt(a, reps=20):
                return time_loop(torch, main, lambda: sp.spmv_rows(a, x, y2, 0, n, x_col0=L.x_col0, x_len=L.x_len, stream=main), reps)
            t_ell = time_fmt(ell)
            extra["ell"] = {"ms": t_ell, "gflops": 2.0 * nnz_local / t_ell / 1e6, "algorithmic_gbs": 340.0 * n / t_ell / 1e6}
            del ell
            csr2 = sp.generate_matrix(sp.GridSpec(nx, ny, nzl * world), row_begin=L.row_range[0],
                                      row_end=L.row_range[1], stream=main)
            vt = sp.compress_values(csr2, min_width=27, stream=main)
            del csr2
            t_vt = time_fmt(vt)
            extra["vt"] = {"ms": t_vt, "gflops": 2.0 * nnz_local / t_vt / 1e6, "algorithmic_gbs": 132.0 * n / t_vt / 1e6}
            del vt
            sp.set_option("pattern_kernel", 1)
            t_gen = time_fmt(pc)
            sp.set_option("pattern_kernel", 0)
            extra["pattern_list1_kernel"] = {"ms": t_gen, "gflops": 2.0 * nnz_local / t_gen / 1e6}
        else:
            del ell
        sampler.stop_flag = True
        sampler.join()

        # ---- end to end through host buffers: H2D x, SpMV, D2H y every step
        Ke = max(3, min(K, 20))
        xh = torch.empty(L.x_len if world > 1 else n, dtype=torch.float64).pin_memory()
        yh = torch.empty(n, dtype=torch.float64).pin_memory()
        if world == 1:
            sp.check(sp.lib.spmvb_vec_download(xh.data_ptr(), x.data_ptr() + 8 * plane, n, main.cuda_stream))
            # the C-ABI host-buffer entry point (spmv(fmt, Vector) -> Vector): matrix resident, x/y cross PCIe
            pc0 = sp.build_slab_pattern(sp, sp.SlabLayout(nx, ny, nzl, 0, 1), None, stream=main)

            def e2e_step():
                sp.check(sp.lib.spmvb_spmv_host(pc0.h, xh.data_ptr(), n, yh.data_ptr()))
        else:
            sp.check(sp.lib.spmvb_vec_download(xh.data_ptr(), x.data_ptr(), L.x_len, main.cuda_stream))

            def e2e_step():
                sp.check(sp.lib.spmvb_vec_upload(x.data_ptr(), xh.data_ptr(), L.x_len, main.cuda_stream))
                slab.spmv(x, y)
                yh.copy_(y, non_blocking=True)
                main.synchronize()
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(Ke):
            e2e_step()
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3
        y_e2e_matches = bool(torch.equal(yh.cuda(), y))
        e2e_pageable = None
        if world == 1:  # the same call with pageable numpy buffers, as a caller that does not pin gets it
            xp, yp = np.array(xh.numpy()), np.empty(n)
            for _ in range(2):
                sp.check(sp.lib.spmvb_spmv_host(pc0.h, xp.ctypes.data, n, yp.ctypes.data))
            t0 = time.perf_counter()
            for _ in range(5):
                sp.check(sp.lib.spmvb_spmv_host(pc0.h, xp.ctypes.data, n, yp.ctypes.data))
            e2e_pageable = (time.perf_counter() - t0) / 5 * 1e3

    # ---- reduce over ranks: time = max, work = sum
    if world > 1:
        t = torch.tensor([ms, e2e_ms, kernel_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e_ms, kernel_ms = t.tolist()
        w = torch.tensor([float(nnz_local), float(n)], dtype=torch.float64, device="cuda")
        dist.all_reduce(w, op=dist.ReduceOp.SUM)
        nnz_total, n_total = w.tolist()
    else:
        nnz_total, n_total = float(nnz_local), float(n)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = measured_peaks()
    value = 2.0 * nnz_total * K / (ms * 1e-3) / 1e9
    alg_bytes = 20.0 * n  # per launch of the dominant kernel: 4 B id + 8 B x + 8 B y per row
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
    ell_roofline = peak * 1e9 * 2.0 * nnz_local / (340.0 * n) / 1e9  # GFLOP/s an uncompressed ELL could reach at peak
    fits = alg_bytes <= 0.8 * l2_bytes
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": make_config(nx, ny, nzl, world),
        "details": {"nnz_per_gpu": nnz_local, "build_seconds": round(build_s, 2),
                    "parallelism": (f"z-slabs x{world}; one-plane x halo by {'NCCL send/recv' if args.exchange == 'nccl' else 'copies from CUDA-IPC-mapped neighbour memory'}; "
                                    f"schedule {args.schedule}; step replayed as a CUDA graph: {graphed or args.exchange == 'p2p'}") if world > 1 else "single GPU",
                    "regime": "L2-resident" if fits else "HBM"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "frac_of_nominal_8000_gbs": achieved / 8000.0,
                     "traffic": ncu_traffic((nx, ny, nzl), family), "peak_source": peak_src,
                     "kernel": KERNEL_NAMES.get(family, str(family)), "kernel_family": family,
                     "kernel_ms": kernel_ms, "algorithmic_bytes_per_launch": alg_bytes,
                     "equivalent_ell_gbs": 340.0 * n / (kernel_ms * 1e-3) / 1e9,
                     "uncompressed_ell_roofline_gflops": ell_roofline,
                     "gflops_over_ell_roofline": (2.0 * nnz_local / (kernel_ms * 1e-3) / 1e9) / ell_roofline},
        "e2e": {"value": 2.0 * nnz_total * Ke / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(8 * (L.x_len if world > 1 else n)), "d2h_bytes_per_step": int(8 * n),
                "steps": Ke, "ms_per_step": e2e_ms / Ke, "call": "spmvb_spmv_host (C-ABI, pinned host x and y)"
                if world == 1 else "H2D x_local, DeviceSlabSpmv.spmv, D2H y per step", "matches_device_result": y_e2e_matches,
                "ms_per_step_pageable_buffers": e2e_pageable},
        "gpu_launches": launches,
        "clocks": sampler.result(),
        "parity": {"max_scaled_deviation_vs_ell": worst_vs_ell, "rows_differing_from_list1_kernel": bits_vs_generic},
        "formats": extra,
    }

    # ---- CPU baseline: the oracle on this box's host cores, bounded sample, rank 0 at N=1 only
    if world == 1 and not args.no_cpu_baseline:
        block, r = cpu_baseline_block(nx, ny, nzl)
        line["cpu_baseline"] = block
        # whole-vector parity against the oracle at full size (bit-exact: summation order kept)
        from oracle import oracle as orc
        yo = np.empty(n)
        orc.spmv_rows(r["pc"], r["x"], yo, 0, n, threads=r["cores"])
        whole(x, y, 0, n)
        main.synchronize()
        yg = y.cpu().numpy()
        line["parity"]["rows_differing_from_cpu_oracle"] = int((yo.view(np.uint64) != yg.view(np.uint64)).sum())
        ids_dev = pc.download("row_pattern")
        line["parity"]["pattern_ids_differing_from_cpu_oracle"] = int((ids_dev != r["pc"].row_pattern).sum())
        # The reference-signature convenience call spmv(const PatternCompressedMatrix&, const Vector&) -> Vector as the C++
        # shim issues it (cpp/spmvcomp_host.cpp:spmv_checked): the struct's arrays uploaded, validated, x in and a fresh y
        # out through pageable host memory, handle destroyed -- per call.  Callers that keep a device handle get `e2e.value`.
        o = r["pc"]
        xs = np.array(r["x"])
        t_sig = []
        for _ in range(3):
            t0 = time.perf_counter()
            d = sp.upload_pattern(o.n, o.table, o.disp_offsets, o.disp_flat, o.ends_flat, o.row_pattern, True)
            sp.check(sp.lib.spmvb_validate(d.h, o.n, None))
            ys = np.empty(n)
            sp.check(sp.lib.spmvb_spmv_host(d.h, xs.ctypes.data, n, ys.ctypes.data))
            del d
            t_sig.append((time.perf_counter() - t0) * 1e3)
        line["e2e"]["ms_per_call_reference_signature"] = min(t_sig)
        line["e2e"]["reference_signature_note"] = ("spmv(fmt, Vector) -> Vector: upload of the struct's arrays (67 MB of ids), validate, "
                                                   "pageable x in / fresh pageable y out, handle destroyed; best of 3")
        line["e2e"]["reference_signature_matches_oracle"] = bool(np.array_equal(ys.view(np.uint64), yo.view(np.uint64)))
        del r, o
    if world == 1 and not args.no_configs:
        torch.cuda.empty_cache()
        line["configs"] = config_blocks(sp, torch, main, peak, l2_bytes)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(args):
    """`python bench.py --gpus N` outside torchrun: start the N ranks (one per GPU) under torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "WARN")
    return subprocess.call(cmd, env=env)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
