"""GEMM1 + GEMM2 of one rank's expert groups at the G120 P=8 LLEP layout (row f6 of VERDICT r1: the
north-star critical-rank layout) through the standalone C-ABI entry, CUDA-event timed per kernel.

    python tools/p8_layout_gemm.py [--rank 0] [--scenario 95:1] [--iters 20] [--mode llep|ep]

Prints one JSON line: rows, groups, per-kernel ms and TFLOP/s over the REAL rows (4·D·H / 2·D·H per row).
Under ncu (-k regex:grouped_gemm) it is the capture target for the P=8 layout."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_2601_17111_b200 import llep as L  # noqa: E402
from synth import workload as W  # noqa: E402
from emulate_p8 import Gemms, rank_groups  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="g120")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--scenario", default="95:1")
    ap.add_argument("--mode", default="llep")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    base = W.CONFIGS[args.config]
    P = args.world
    sh = W.LayerShape(base.n_experts, base.top_k, base.d_model, base.d_ff, base.tokens_per_rank, P)
    pct, nhot = (int(v) for v in args.scenario.split(":"))
    hot = None if pct == 0 else pct
    cnt = W.slot_counts(sh.n_experts, sh.tokens_per_rank * sh.top_k, hot, nhot)
    plan = L.plan_host((cnt * P).tolist(), P, 1.0, 1024, 1.3, ep=(args.mode == "ep"))
    rows = rank_groups(plan, args.rank, sh.experts_per_rank)
    g = Gemms(rows, sh.d_model, sh.d_ff)
    D, H = sh.d_model, sh.d_ff
    for _ in range(3):
        g.run_ms(1)
    # no host synchronisation inside the loop: the host-side preparation of each launch (group table,
    # schedule, tensor maps) runs ahead of the GPU instead of being timed as idle time
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.iters)]
    for e in ev:
        e[0].record()
        L.grouped_gemm(0, g.x, g.w13, g.groups, H, out=g.act, pair=True)
        e[1].record()
        L.grouped_gemm(1, g.act, g.w2, g.groups, D, gate=g.gate, out=g.y, pair=True)
        e[2].record()
    torch.cuda.synchronize()
    t1 = sum(e[0].elapsed_time(e[1]) for e in ev[1:]) / (args.iters - 1)
    t2 = sum(e[1].elapsed_time(e[2]) for e in ev[1:]) / (args.iters - 1)
    n = sum(rows)
    print(json.dumps({"config": args.config, "world": P, "rank": args.rank, "scenario": args.scenario,
                      "mode": args.mode, "rows": n, "groups": len(rows), "group_rows": rows[:20],
                      "gemm1_ms": t1, "gemm2_ms": t2, "gemm1_tflops": 4 * D * H * n / t1 / 1e9,
                      "gemm2_tflops": 2 * D * H * n / t2 / 1e9,
                      "both_tflops": 6 * D * H * n / (t1 + t2) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
