"""Backward row GEMMs (llep_gemm_bwd kind 0, CTA pairs: dA0 = dO·W_down, dX = dGU·W13) on the G120
P=8 critical-rank layout or the P=1 layout: time per launch (CUDA events, median of 10 after 0.4 s of
warm-up) and TFLOP/s over the real rows.  Under ncu (-k regex:gemm_bwd_pair) it is the capture target.
    python tools/bwd_rows_bench.py [p8|both|hot|cold] [kdim] [nout]     (dA0: 2880 2880, dX: 5760 2880)"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17111_b200 import llep as L  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "p8"
kdim = int(sys.argv[2]) if len(sys.argv) > 2 else 2880
nout = int(sys.argv[3]) if len(sys.argv) > 3 else 2880
sizes = {"both": [124518] + [52] * 127, "p8": [124832] + [416] * 15, "hot": [124832], "cold": [416] * 15}[which]
groups, rb = [], 0
for i, n in enumerate(sizes):
    groups.append((i, rb, n))
    rb += (n + 255) // 256 * 256
torch.manual_seed(0)
a = torch.randn(rb, kdim, device="cuda").to(torch.bfloat16)
w = (torch.randn(len(sizes), kdim, nout, device="cuda") / kdim ** 0.5).to(torch.bfloat16)
out = torch.zeros(rb, nout, device="cuda", dtype=torch.bfloat16)
t0 = time.perf_counter()
while time.perf_counter() - t0 < 0.4:
    L.gemm_bwd(0, a, w, groups, nout, kdim, len(sizes), out=out, pair=True)
    torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        L.gemm_bwd(0, a, w, groups, nout, kdim, len(sizes), out=out, pair=True)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 4)
ms = statistics.median(ts)
flops = 2.0 * kdim * nout * sum(sizes)
print(f"{which} kdim={kdim} nout={nout}: {ms:.3f} ms, {flops / ms / 1e9:.0f} TFLOP/s", flush=True)
