"""Weight-gradient GEMM (llep_gemm_bwd kind 1, CTA pairs) on G120-P1-like group layouts: time per
launch (CUDA events, median of 10 after 0.4 s of back-to-back warm-up) and the output write rate.
    python tools/wgrad_bench.py [hot|small|both|p8] [mdim] [nout] [--1cta]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17111_b200 import llep as L  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
mdim = int(sys.argv[2]) if len(sys.argv) > 2 else 2880
nout = int(sys.argv[3]) if len(sys.argv) > 3 else 2880
pair = "--1cta" not in sys.argv
sizes = {"hot": [124518], "small": [52] * 127, "both": [124518] + [52] * 127,
         "p8": [124832] + [416] * 15}[which]   # p8: the G120 P=8 LLEP critical-rank layout
groups, rb = [], 0
for i, n in enumerate(sizes):
    groups.append((i, rb, n))
    rb += (n + 255) // 256 * 256
torch.manual_seed(0)
a = torch.randn(rb, mdim, device="cuda").to(torch.bfloat16)
b = torch.randn(rb, nout, device="cuda").to(torch.bfloat16)
for (i, r0, n) in groups:
    a[r0 + n:r0 + (n + 255) // 256 * 256] = 0
    b[r0 + n:r0 + (n + 255) // 256 * 256] = 0
out = torch.empty(len(groups), mdim, nout, device="cuda")
import time  # noqa: E402
t0 = time.perf_counter()
while time.perf_counter() - t0 < 0.4:          # steady state: clocks settle under the power cap
    L.gemm_bwd(1, a, b, groups, nout, mdim, len(groups), out=out, pair=pair)
    torch.cuda.synchronize()
ts = []
for _ in range(10):   # 4 back-to-back launches per event pair: the host-side preparation overlaps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        L.gemm_bwd(1, a, b, groups, nout, mdim, len(groups), out=out, pair=pair)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 4)
ms = statistics.median(ts)
flops = 2.0 * mdim * nout * sum(sizes)
wbytes = len(groups) * mdim * nout * 4
import hashlib  # noqa: E402
digest = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12]   # A/B variants must agree bitwise
print(f"{which} mdim={mdim} nout={nout} pair={pair}: {ms:.3f} ms, {flops / ms / 1e9:.0f} TFLOP/s, "
      f"output {wbytes / 1e9:.2f} GB -> {wbytes / ms / 1e6:.0f} GB/s, sha1 {digest}", flush=True)
