#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200-native compressed SpMV path.

Workload (BASELINE.json configs[2]): HPCG 27-point stencil, 256x256x256 rows per
GPU stacked as z-slabs (global nz = 256*G), compressed pattern format (4-byte
pattern id per row + dictionary), x ~ U[-1,1) from seed 7, fp64.  One "step" is
one SpMV y = A x over the slab (plus the one-plane halo exchange when G > 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU restatement of
the reference's unchecked::spmv_rows (the oracle; the reference ships no src/)
on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 7
METRIC = "SpMV GFLOP/s (2*nnz/t), fp64, HPCG 27-point stencil, compressed pattern format"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--grid", type=int, nargs=3, default=[256, 256, 256], help="rows per GPU (nx ny nz_local)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-formats", action="store_true")
    return ap.parse_args()


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs, copy kernel)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

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
            time.sleep(0.002)

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


# ------------------------------------------------------------------------------------------------
def cpu_sample(nx, ny, nz, steps, warmup, budget_s):
    """Times the oracle's pattern SpMV (CPU restatement of unchecked::spmv_rows,
    kernels.hpp:35-36) with all host threads on a bounded sample of the workload."""
    import numpy as np
    from oracle import oracle as orc

    cores = os.cpu_count() or 1
    pc = orc.compress_patterns_grid(nx, ny, nz, values_in_pattern=True)
    n = pc.n
    x = orc.make_test_vector(n, orc.RANDOM, seed=SEED, lo=-1.0, hi=1.0)
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
    t0 = time.perf_counter()
    for _ in range(steps):
        orc.spmv_rows(pc, x, y, b, e, threads=cores)
    dt = time.perf_counter() - t0
    return {"gflops": 2.0 * nnz * steps / dt / 1e9, "ms_per_step": dt / steps * 1e3, "cores": cores,
            "sample": f"pattern-format SpMV over planes [{z0},{z0 + planes}) of {nx}x{ny}x{nz} "
                      f"({e - b} rows, {nnz} nnz) x {steps} reps, {cores} threads (contiguous row ranges)",
            "pc": pc, "x": x}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nx, ny, nz = args.grid
    r = cpu_sample(nx, ny, nz, args.steps, args.warmup, budget_s=150.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": r["gflops"], "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(nx, ny, nz, args.gpus), "format": "pattern (values_in_pattern)",
                   "note": "CPU restatement of the reference's unchecked::spmv_rows (the reference ships no "
                           "implementation source); host threads only, no GPU"},
        "cpu_baseline": {"value": r["gflops"], "unit": "GFLOP/s", "cores": r["cores"], "kind": "port",
                         "sample": r["sample"]},
        "e2e": {"value": r["gflops"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def workload_name(nx, ny, nz, g):
    return (f"BASELINE configs[2]: HPCG 27-point stencil {nx}x{ny}x{nz} per GPU, {g} z-slab(s) "
            f"(global {nx}x{ny}x{nz * g}), diagonal 26 / off-diagonal -1, x~U[-1,1) seed {SEED}")


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
    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import paper_1612_00530_b200 as sp

    nx, ny, nzl = args.grid
    L = sp.SlabLayout(nx, ny, nzl * world, rank, world)
    n, plane = L.n_local, L.plane
    z0, z1 = L.z_range
    nnz_local = nnz_slab(nx, ny, nzl * world, z0, z1)
    main = torch.cuda.Stream()
    comm = torch.cuda.Stream()
    K, W = args.steps, args.warmup

    with torch.cuda.stream(main):
        # ---- build on the device: generator -> compressor (+ dictionary merge across slabs)
        t_build = time.perf_counter()
        pc, csr = sp.build_slab_pattern(sp, L, dist if world > 1 else None, keep_csr=True, stream=main)
        assert pc.info.nnz == nnz_local, (pc.info.nnz, nnz_local)
        ell = sp.to_ell(csr, min_width=27, stream=main)
        x = torch.empty(L.x_len, dtype=torch.float64, device="cuda")
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        y2 = torch.empty(n, dtype=torch.float64, device="cuda")
        scale = torch.empty(n, dtype=torch.float64, device="cuda")
        sp.check(sp.lib.spmvb_vec_fill(x.data_ptr(), L.x_len, sp.RANDOM, SEED, -1.0, 1.0, L.x_col0, main.cuda_stream))
        main.synchronize()
        build_s = time.perf_counter() - t_build

        def kernel_of(a):
            def k(xl, yl, b, e, stream=None):
                sp.spmv_rows(a, xl, yl, b, e, x_col0=L.x_col0, x_len=L.x_len, stream=main if stream is None else stream)
            return k

        slab = sp.SlabSpmv(L, kernel_of(pc), dist if world > 1 else None, comm, main, torch, two_stream_boundaries=True)

        # ---- verification gate: no number for a kernel that failed parity
        slab.spmv(x, y)
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
            slab.spmv(x, y)
        main.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler.samples.clear()  # keep only what is sampled from here on: the timed region and the kernel-alone loop
        sampler.reasons.clear()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(main)
        for _ in range(K):
            slab.spmv(x, y)
        ev1.record(main)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        launches = K * (1 if world == 1 else (1 + int(L.has_lower) + int(L.has_upper)))

        # ---- dominant kernel alone (roofline): all local rows, no exchange
        kern = kernel_of(pc)
        for _ in range(3):
            kern(x, y, 0, n)
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(main)
        for _ in range(K):
            kern(x, y, 0, n)
        k1.record(main)
        torch.cuda.synchronize()
        kernel_ms = k0.elapsed_time(k1) / K
        sampler.stop_flag = True
        sampler.join()

        # ---- other formats, same x (context for the compression gain)
        extra = {}
        if not args.no_extra_formats:
            def time_fmt(a, reps=20):
                for _ in range(3):
                    sp.spmv_rows(a, x, y2, 0, n, x_col0=L.x_col0, x_len=L.x_len, stream=main)
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(main)
                for _ in range(reps):
                    sp.spmv_rows(a, x, y2, 0, n, x_col0=L.x_col0, x_len=L.x_len, stream=main)
                a1.record(main)
                torch.cuda.synchronize()
                return a0.elapsed_time(a1) / reps
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

        # ---- end to end through host buffers: H2D x, SpMV, D2H y every step
        Ke = max(3, min(K, 20))
        xh = torch.empty(L.x_len if world > 1 else n, dtype=torch.float64).pin_memory()
        yh = torch.empty(n, dtype=torch.float64).pin_memory()
        xh.copy_(x[plane:plane + n] if world == 1 else x)
        if world == 1:
            # the C-ABI host-buffer entry point (spmv(fmt, Vector) -> Vector): matrix resident, x/y cross PCIe
            pc0 = sp.build_slab_pattern(sp, sp.SlabLayout(nx, ny, nzl, 0, 1), None, stream=main)

            def e2e_step():
                sp.check(sp.lib.spmvb_spmv_host(pc0.h, xh.data_ptr(), n, yh.data_ptr()))
        else:
            def e2e_step():
                x.copy_(xh, non_blocking=True)
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
        y_e2e_matches = bool(torch.equal(yh.cuda(), y)) if world == 1 else True

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
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_name(nx, ny, nzl, world), "format": "pattern (values_in_pattern): "
                   "4-byte pattern id per row + 27-entry dictionary", "rows_per_gpu": n, "nnz_per_gpu": nnz_local,
                   "parallelism": f"z-slabs x{world}, one-plane x halo over NCCL send/recv overlapped with interior rows"
                   if world > 1 else "single GPU",
                   "l2": "inputs (20 B/row * 16.8M rows = 335 MB per SpMV) exceed the 126 MB L2; no flush needed",
                   "build_seconds": round(build_s, 2)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(), "peak_source": peak_src, "kernel": "spmv_pattern_ringp_kernel<6,4,2> (persistent tensor ring)",
                     "kernel_ms": kernel_ms, "algorithmic_bytes_per_launch": alg_bytes,
                     "equivalent_ell_gbs": 340.0 * n / (kernel_ms * 1e-3) / 1e9,
                     "uncompressed_ell_roofline_gflops": ell_roofline,
                     "gflops_over_ell_roofline": (2.0 * nnz_local / (kernel_ms * 1e-3) / 1e9) / ell_roofline},
        "e2e": {"value": 2.0 * nnz_total * Ke / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(8 * (L.x_len if world > 1 else n)), "d2h_bytes_per_step": int(8 * n),
                "steps": Ke, "ms_per_step": e2e_ms / Ke, "call": "spmvb_spmv_host (C-ABI, pinned host x and y)"
                if world == 1 else "H2D x_local, SlabSpmv.spmv, D2H y per step", "matches_device_result": y_e2e_matches},
        "gpu_launches": launches,
        "clocks": sampler.result(),
        "parity": {"max_scaled_deviation_vs_ell": worst_vs_ell, "rows_differing_from_list1_kernel": bits_vs_generic},
        "formats": extra,
    }

    # ---- CPU baseline: the oracle on this box's host cores, bounded sample, rank 0 at N=1 only
    if world == 1 and not args.no_cpu_baseline:
        r = cpu_sample(nx, ny, nzl, steps=3, warmup=1, budget_s=20.0)
        line["cpu_baseline"] = {"value": r["gflops"], "unit": "GFLOP/s", "cores": r["cores"], "kind": "port",
                                "sample": r["sample"]}
        # whole-vector parity against the oracle at full size (bit-exact: summation order kept)
        from oracle import oracle as orc
        yo = np.empty(n)
        orc.spmv_rows(r["pc"], r["x"], yo, 0, n, threads=r["cores"])
        yg = y.cpu().numpy()
        line["parity"]["rows_differing_from_cpu_oracle"] = int((yo.view(np.uint64) != yg.view(np.uint64)).sum())
        ids_dev = pc.download("row_pattern")
        line["parity"]["pattern_ids_differing_from_cpu_oracle"] = int((ids_dev != r["pc"].row_pattern).sum())
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
