"""Steady-state A/B of the forward grouped GEMMs (GEMM1 + GEMM2) on two group layouts with the same
real rows, strictly alternating iterations (both arms see the same power-capped clock), median.

    python tools/layout_ab.py g120p1 dense      # G120 at P=1 (1 hot + 127 cold experts) vs one group
"""
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from emulate_p8 import Gemms, L  # noqa: E402

LAYOUTS = {
    "g120p1": [124518] + [52] * 77 + [51] * 50,
    "dense": [131072],
    "hot": [124518],
    "cold": [52] * 77 + [51] * 50,
    "g120p8": [124464] + [413] * 16,
    "uniform16": [8192] * 16,
    "cold128": [128] * 127,      # same experts, every cold group filling its M=128 pair tile
    "cold256": [256] * 127,      # ... a full M=256 pair tile
    "cold64g": [52] * 64,        # half the cold experts
}


def batch_ms(g, reps=6):
    """Per-iteration GPU time of `reps` back-to-back GEMM1+GEMM2 pairs between one event pair: the
    host-side preparation of llep_grouped_gemm (group table, schedule, tensor maps) overlaps the
    previous launches, so only the first one is exposed (amortised over reps)."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        L.grouped_gemm(0, g.x, g.w13, g.groups, g.H, out=g.act, pair=True)
        L.grouped_gemm(1, g.act, g.w2, g.groups, g.D, gate=g.gate, out=g.y, pair=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    a, b = sys.argv[1], sys.argv[2]
    D = H = 2880
    g = {k: Gemms(LAYOUTS[k], D, H) for k in (a, b)}
    for k in g:
        g[k].run_ms()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.3:
        g[a].run_ms()
    ms = {a: [], b: []}
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 1.5:
        for k in (a, b):
            ms[k].append(batch_ms(g[k]))
    res = {k: {"rows": sum(LAYOUTS[k]), "groups": len(LAYOUTS[k]), "gemm_ms": statistics.median(v),
               "tflops": 6.0 * D * H * sum(LAYOUTS[k]) / statistics.median(v) / 1e9, "iters": len(v)}
           for k, v in ms.items()}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
