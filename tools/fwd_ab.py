"""In-situ A/B of an environment switch read per launch by the library (e.g. LLEP_GEMM_PREFETCH) on
the real layer forward (llep_prepare + llep_moe_forward, device-side layout), one process, strictly
alternating batches so both arms see the same power-capped clock; median per-step time.

    python tools/fwd_ab.py LLEP_GEMM_PREFETCH 0 1 [--config g120] [--hot 95] [--secs 3]
"""
import argparse
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_17111_b200 import llep as L  # noqa: E402
from synth import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("var")
    ap.add_argument("a")
    ap.add_argument("b")
    ap.add_argument("--config", default="g120")
    ap.add_argument("--hot", type=int, default=95)
    ap.add_argument("--secs", type=float, default=3.0)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--train", action="store_true",
                    help="time a training step: prepare + forward_train + backward from the saved [g|u]")
    args = ap.parse_args()
    base = W.CONFIGS[args.config]
    sh = W.LayerShape(base.n_experts, base.top_k, base.d_model, base.d_ff, base.tokens_per_rank, 1)
    dev = "cuda:0"
    seed = 2601017111
    ids = torch.from_numpy(W.routing_ids(sh, 0, args.hot or None, 1, seed)).to(dev)
    gates = torch.from_numpy(W.gate_weights(sh.tokens_per_rank, sh.top_k, 0, seed)).to(dev)
    x = W.tokens_torch(sh.tokens_per_rank, sh.d_model, 0, dev, seed)
    w13, w2 = W.expert_weights_torch(range(sh.n_experts), sh.d_model, sh.d_ff, dev, seed)
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, 1, 0, 0, sh.tokens_per_rank)
    out = torch.empty_like(x)
    plan_buf = torch.empty(L.plan_bytes(sh.n_experts, 1), dtype=torch.uint8, device=dev)
    outs = {}
    if args.train:
        ctx.enable_backward()
        dout = W.tokens_torch(sh.tokens_per_rank, sh.d_model, 1000, dev, seed)
        M, D, H = sh.experts_per_rank, sh.d_model, sh.d_ff
        dx, dg = torch.empty_like(x), torch.empty(ids.shape, dtype=torch.float32, device=dev)
        dw13 = torch.empty((M, 2 * H, D), dtype=torch.float32, device=dev)
        dw2 = torch.empty((M, D, H), dtype=torch.float32, device=dev)
        gu = [None]

    def batch(val):
        os.environ[args.var] = val
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            plan, req = ctx.prepare(ids, plan_out=plan_buf)
            if args.train:
                if gu[0] is None:
                    gu[0] = torch.empty((int(req.rows_needed), 2 * sh.d_ff), dtype=torch.bfloat16, device=dev)
                ctx.forward_train(x, ids, gates, w13, w2, plan, out, gu[0])
                ctx.backward(x, ids, gates, dout, w13, w2, plan, dx, dg, dw13, dw2, gu=gu[0])
            else:
                ctx.forward(x, ids, gates, w13, w2, plan, out)
        e1.record()
        torch.cuda.synchronize()
        outs[val] = (dx if args.train else out).clone()
        return e0.elapsed_time(e1) / args.reps

    for v in (args.a, args.b):
        batch(v)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.5:
        batch(args.a)
    ms = {args.a: [], args.b: []}
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < args.secs:
        for v in (args.a, args.b):
            ms[v].append(batch(v))
    res = {"var": args.var, "config": args.config, "hot": args.hot,
           "same_output": bool(torch.equal(outs[args.a], outs[args.b]))}
    for v in (args.a, args.b):
        med = statistics.median(ms[v])
        res[v] = {"ms_per_step": med, "tokens_s": sh.tokens_per_rank / med * 1e3, "iters": len(ms[v])}
    res["speedup_b_over_a"] = res[args.a]["ms_per_step"] / res[args.b]["ms_per_step"]
    print(json.dumps(res), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
