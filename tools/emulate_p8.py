"""Critical-rank emulation of the 8-GPU comparison on one B200.

For a scenario of the G120 layer (N=128, K=4, D=H=2880, 32K tokens per rank, P=8) the plans of all
ranks are computed from the synthetic routing (host planner, bit-identical to the device one); for
standard EP and for LLEP the most loaded rank's expert groups (rows per expert, in the layout
kernel's order) are built and that rank's two grouped GEMMs are timed on this GPU through the C ABI
(2-CTA kernels, CUDA events; steady state: each mode runs back to back for >= 150 ms per round,
rounds alternate, median of all iterations).  The GEMMs are ~93 % of a layer step at P=1;
dispatch / combine / weight-broadcast costs over NVLink are NOT measured here.

    python tools/emulate_p8.py [--scenarios 95:1,80:1,...] [--reps 5]
"""
import argparse
import json
import os
import statistics
import sys
import time

import math

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_17111_b200 import llep as L  # noqa: E402
from synth import workload as W  # noqa: E402

NVLINK = 900e9   # NVLink 5, per direction (modelled link time only)


def rank_groups(plan, rank, M):
    rows = []
    for pass_ in (0, 1):
        for e, chunks in enumerate(plan.chunks):
            native = e // M == rank
            if native != (pass_ == 0):
                continue
            r = sum(t - s for (d, s, t) in chunks if d == rank)
            if r:
                rows.append(r)
    return rows


def link_seconds(plan, cnt, D, H, M, P=8, aligned=True):
    """Modelled NVLink time of one layer: dispatch + combine rows and the weight broadcast.  Every rank
    has the same counts cnt; source blocks in the library's token order (chunk-aligned R11' by default:
    an expert with > 1 chunk lists its chunk devices in plan order first, then the other ranks)."""
    egress = np.zeros(P)
    ingress = np.zeros(P)
    for e, chunks in enumerate(plan.chunks):
        c = int(cnt[e])
        srcs = list(range(P))
        if aligned and len(chunks) > 1:
            first = []
            for (d, _s, _t) in chunks:
                if d not in first:
                    first.append(d)
            srcs = first + [q for q in range(P) if q not in first]
        pos = {p: i for i, p in enumerate(srcs)}   # source p's block: global [pos·c, (pos+1)·c)
        for (d, s, t) in chunks:
            for p in range(P):
                n = max(0, min(t, (pos[p] + 1) * c) - max(s, pos[p] * c))
                if n and p != d:
                    egress[p] += n * (2 * D + 4 + 2 * D)
                    ingress[d] += n * (2 * D + 4 + 2 * D)
    t_rows = max(egress.max(), ingress.max()) / NVLINK
    reps = {}
    for (e, src, dst) in plan.transfers:
        reps.setdefault(e, []).append(dst)
    wsrc = np.zeros(P)
    for e, ds in reps.items():
        wsrc[e // M] += math.ceil(math.log2(len(ds) + 1)) * 6 * D * H
    return t_rows + wsrc.max() / NVLINK


class Gemms:
    """The critical rank's grouped GEMM1 + GEMM2 on synthetic data (values do not matter for time)."""

    def __init__(self, rows, D, H):
        groups, rb = [], 0
        for i, n in enumerate(rows):
            groups.append((i, rb, n))
            rb += (n + 255) // 256 * 256
        E = len(rows)
        self.groups, self.D, self.H = groups, D, H
        self.x = torch.randn(rb, D, device="cuda").to(torch.bfloat16)
        self.w13 = (torch.randn(E, 2 * H, D, device="cuda") / D ** 0.5).to(torch.bfloat16)
        self.w2 = (torch.randn(E, D, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
        self.act = torch.empty(rb, H, device="cuda", dtype=torch.bfloat16)
        self.y = torch.empty(rb, D, device="cuda", dtype=torch.bfloat16)
        self.gate = torch.rand(rb, device="cuda")

    def run_ms(self, reps=3):
        """Per-iteration GPU time of `reps` back-to-back GEMM1 + GEMM2 pairs between one event pair:
        the host-side preparation of llep_grouped_gemm (group table, schedule, tensor maps) then
        overlaps the previous launches instead of being timed as GPU idle."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            L.grouped_gemm(0, self.x, self.w13, self.groups, self.H, out=self.act, pair=True)
            L.grouped_gemm(1, self.act, self.w2, self.groups, self.D, gate=self.gate, out=self.y, pair=True)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="g120")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--scenarios", default="95:1,80:1,50:1,30:1,95:4,95:16,0:0")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    base = W.CONFIGS[args.config]
    P = args.world
    sh = W.LayerShape(base.n_experts, base.top_k, base.d_model, base.d_ff, base.tokens_per_rank, P)
    M = sh.experts_per_rank
    out = []
    for sc in args.scenarios.split(","):
        pct, nhot = (int(v) for v in sc.split(":"))
        hot = None if pct == 0 else pct
        cnt = W.slot_counts(sh.n_experts, sh.tokens_per_rank * sh.top_k, hot, nhot)
        loads = (cnt * P).tolist()   # every rank draws the same per-expert slot counts (exact multiset)
        res = {"config": args.config, "world": P, "scenario": W.scenario_name(hot, nhot)}
        g = {}
        for mode in ("ep", "llep"):
            plan = L.plan_host(loads, P, 1.0, 1024, 1.3, ep=(mode == "ep"))
            per_rank = [sum(rank_groups(plan, r, M)) for r in range(P)]
            crit = int(np.argmax(per_rank))
            rows = rank_groups(plan, crit, M)
            g[mode] = Gemms(rows, sh.d_model, sh.d_ff)
            res[mode] = {"critical_rank": crit, "rows": int(sum(rows)), "groups": len(rows),
                         "transfers": len(plan.transfers), "fallback": plan.fallback,
                         "link_ms_modelled": 1e3 * link_seconds(plan, cnt, sh.d_model, sh.d_ff, M, P), "ms": []}
        for m in ("ep", "llep"):
            g[m].run_ms()                      # warm-up
        # steady state under the power cap: 0.3 s of back-to-back warm-up, then EP and LLEP iterations
        # strictly alternating for >= 0.3 s per rep (both arms see the same clock / thermal state),
        # median over all CUDA-event-timed iterations
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 0.3:
            g["llep"].run_ms()
        for _ in range(args.reps):
            t0, n = time.perf_counter(), 0
            while n < 3 or time.perf_counter() - t0 < 0.3:
                for m in ("ep", "llep"):
                    res[m]["ms"].append(g[m].run_ms())
                n += 1
        for m in ("ep", "llep"):
            res[m]["iters"] = len(res[m]["ms"])
            res[m]["gemm_ms"] = statistics.median(res[m].pop("ms"))
        del g
        torch.cuda.empty_cache()
        res["gemm_speedup"] = res["ep"]["gemm_ms"] / res["llep"]["gemm_ms"]
        res["row_bound"] = res["ep"]["rows"] / res["llep"]["rows"]
        res["modelled_layer_speedup"] = ((res["ep"]["gemm_ms"] + res["ep"]["link_ms_modelled"]) /
                                         (res["llep"]["gemm_ms"] + res["llep"]["link_ms_modelled"]))
        print(json.dumps(res), flush=True)
        out.append(res)
    return out


if __name__ == "__main__":
    main()
