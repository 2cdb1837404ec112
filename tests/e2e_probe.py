"""Exploratory: end-to-end host-buffer SpMV time vs the number of pipeline chunks (GPU box)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1612_00530_b200 as sp
n1 = 256
m = sp.generate_matrix(sp.GridSpec(n1, n1, n1))
pc = sp.compress_patterns(m, True)
del m
n = pc.info.n
x = torch.empty(n, dtype=torch.float64).pin_memory()
y = torch.empty(n, dtype=torch.float64).pin_memory()
x.uniform_(-1, 1)
import ctypes as C
def run():
    sp.check(sp.lib.spmvb_spmv_host(pc.h, C.c_void_p(x.data_ptr()), n, C.c_void_p(y.data_ptr())))
for chunks in (1, 4, 8, 16, 32, 64):
    sp.set_option("host_chunks", chunks)
    for _ in range(3): run()
    t0 = time.perf_counter()
    for _ in range(20): run()
    dt = (time.perf_counter() - t0) / 20
    print(f"chunks {chunks:3d}: {dt*1e3:.3f} ms per call")

# the 16 chunk kernels alone (device-resident x, y), one stream
xd = torch.empty(n, dtype=torch.float64, device="cuda"); yd = torch.empty(n, dtype=torch.float64, device="cuda")
xd.uniform_(-1, 1)
per = n // 16
def chunks16():
    for k in range(16):
        sp.spmv_rows(pc, xd, yd, k * per, (k + 1) * per)
for _ in range(3): chunks16()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(20): chunks16()
e1.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"16 chunk kernels: GPU {e0.elapsed_time(e1)/20:.3f} ms per sweep, CPU enqueue {(t1-t0)/20*1e3:.3f} ms per sweep")

# the same pipeline driven from Python: H2D chunk -> kernel chunk -> D2H chunk on three streams
s_in, s_run, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
plane = n1 * n1
for chunks in (8, 16):
    per = n // chunks
    ev_in = [torch.cuda.Event() for _ in range(chunks)]
    ev_run = [torch.cuda.Event() for _ in range(chunks)]
    def pipe():
        sent = 0
        for k in range(chunks):
            r0, r1 = k * per, (k + 1) * per
            need = min(n, r1 + plane + n1 + 1)
            with torch.cuda.stream(s_in):
                if need > sent:
                    xd[sent:need].copy_(x[sent:need], non_blocking=True)
                    sent = need
                ev_in[k].record(s_in)
            s_run.wait_event(ev_in[k])
            sp.spmv_rows(pc, xd, yd, r0, r1, stream=s_run)
            ev_run[k].record(s_run)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_run[k])
                y[r0:r1].copy_(yd[r0:r1], non_blocking=True)
        s_out.synchronize()
    for _ in range(3): pipe()
    t0 = time.perf_counter()
    for _ in range(20): pipe()
    print(f"python-driven pipeline, {chunks} chunks: {(time.perf_counter()-t0)/20*1e3:.3f} ms per call")

def make_pipe(chunks, kind):
    per = n // chunks
    ev_in = [torch.cuda.Event() for _ in range(chunks)]
    ev_run = [torch.cuda.Event() for _ in range(chunks)]
    def pipe():
        sent = 0
        for k in range(chunks):
            r0, r1 = k * per, (k + 1) * per
            need = min(n, r1 + plane + n1 + 1)
            with torch.cuda.stream(s_in):
                if need > sent:
                    xd[sent:need].copy_(x[sent:need], non_blocking=True)
                    sent = need
                ev_in[k].record(s_in)
            s_run.wait_event(ev_in[k])
            if kind == "copy-kernel":
                with torch.cuda.stream(s_run):
                    yd[r0:r1].copy_(xd[r0:r1])
            elif kind == "spmv":
                sp.spmv_rows(pc, xd, yd, r0, r1, stream=s_run)
            elif kind == "spmv-box3":
                sp.set_option("box_march", 3)
                sp.spmv_rows(pc, xd, yd, r0, r1, stream=s_run)
                sp.set_option("box_march", 0)
            ev_run[k].record(s_run)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_run[k])
                y[r0:r1].copy_(yd[r0:r1], non_blocking=True)
        s_out.synchronize()
    return pipe
for kind in ("none", "copy-kernel", "spmv", "spmv-box3"):
    pipe = make_pipe(16, kind)
    for _ in range(3): pipe()
    t0 = time.perf_counter()
    for _ in range(20): pipe()
    print(f"pipeline 16 chunks, kernel = {kind:12s}: {(time.perf_counter()-t0)/20*1e3:.3f} ms per call")

def make_pipe2(chunks, hop, shifted):
    per = n // chunks
    ev_in = [torch.cuda.Event() for _ in range(chunks)]
    ev_run = [torch.cuda.Event() for _ in range(chunks)]
    def pipe():
        sent = 0
        for k in range(chunks):
            r0, r1 = k * per, (k + 1) * per
            need = min(n, r1 + plane + n1 + 1) if shifted else r1
            with torch.cuda.stream(s_in):
                if need > sent:
                    xd[sent:need].copy_(x[sent:need], non_blocking=True)
                    sent = need
                ev_in[k].record(s_in)
            if hop:
                s_run.wait_event(ev_in[k])
                ev_run[k].record(s_run)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_run[k] if hop else ev_in[k])
                y[r0:r1].copy_(yd[r0:r1], non_blocking=True)
        s_out.synchronize()
    return pipe
for hop in (False, True):
    for shifted in (False, True):
        pipe = make_pipe2(16, hop, shifted)
        for _ in range(3): pipe()
        t0 = time.perf_counter()
        for _ in range(20): pipe()
        print(f"copy-only pipeline hop={hop} shifted={shifted}: {(time.perf_counter()-t0)/20*1e3:.3f} ms per call")
