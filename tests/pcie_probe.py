"""Exploratory: PCIe rates on the GPU box -- whole-vector copies, and the chunked duplex pipeline without any kernel."""
import time
import torch
n = 16777216
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
def h2d():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D 134MB {a:.3f} ms ({0.134217728/a*1e3:.1f} GB/s)  D2H {b:.3f} ms ({0.134217728/b*1e3:.1f} GB/s)  both concurrently {c:.3f} ms")
for chunks in (4, 8, 16, 32):
    per = n // chunks
    evs = [torch.cuda.Event() for _ in range(chunks)]
    def pipe():
        for k in range(chunks):
            with torch.cuda.stream(s1):
                d[k * per:(k + 1) * per].copy_(h[k * per:(k + 1) * per], non_blocking=True)
                evs[k].record(s1)
            with torch.cuda.stream(s2):
                s2.wait_event(evs[k])
                h2[k * per:(k + 1) * per].copy_(d[k * per:(k + 1) * per], non_blocking=True)
    print(f"chunked duplex pipeline, {chunks:2d} chunks, no kernel: {t(pipe):.3f} ms")
