"""Probe PCIe copy concurrency: H2D alone, D2H alone, both at once, both under a busy GPU."""
import torch, time
n = 32768 * 2880
xh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
oh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
xd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
od = torch.empty(n, dtype=torch.bfloat16, device="cuda")
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
def h2d():
    with torch.cuda.stream(s1): xd.copy_(xh, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): oh.copy_(od, non_blocking=True)
def both(): h2d(); d2h()
def gemm():
    with torch.cuda.stream(s3):
        for _ in range(4): a @ a
def all3(): gemm(); h2d(); d2h()
print(f"bytes {n*2/1e6:.0f} MB; h2d {t(h2d):.2f} ms  d2h {t(d2h):.2f} ms  both {t(both):.2f} ms  gemm {t(gemm):.2f} ms  gemm+both {t(all3):.2f} ms")
