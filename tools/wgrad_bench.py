"""Weight-gradient GEMM (llep_gemm_bwd kind 1) on G120-P1-like group layouts, for ncu A/B.
    python tools/wgrad_bench.py [hot|small|both] [mdim] [nout]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17111_b200 import llep as L
which = sys.argv[1] if len(sys.argv) > 1 else "both"
mdim = int(sys.argv[2]) if len(sys.argv) > 2 else 2880
nout = int(sys.argv[3]) if len(sys.argv) > 3 else 2880
sizes = {"hot": [124518], "small": [52] * 127, "both": [124518] + [52] * 127}[which]
groups, rb = [], 0
for i, n in enumerate(sizes):
    groups.append((i, rb, n))
    rb += (n + 255) // 256 * 256
a = torch.randn(rb, mdim, device="cuda").to(torch.bfloat16)
b = torch.randn(rb, nout, device="cuda").to(torch.bfloat16)
for (i, r0, n) in groups:
    a[r0 + n:r0 + (n + 255) // 256 * 256] = 0
    b[r0 + n:r0 + (n + 255) // 256 * 256] = 0
out = torch.empty(len(groups), mdim, nout, device="cuda")
for _ in range(3):
    L.gemm_bwd(1, a, b, groups, nout, mdim, len(groups), out=out)
torch.cuda.synchronize()
