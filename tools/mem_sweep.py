"""Measured peak memory per GPU at P = 2/4/8 (BASELINE metric "peak GB/GPU ... LLEP vs EP"), on one B200.

P ranks run as P processes sharing cuda:0 (CUDA-IPC arenas, gloo for plumbing, as in the multi-rank
tests).  Every rank holds exactly what it would hold on its own GPU -- its M native experts, its
tokens, ids, gates, output, and the library context (symmetric arena, scratch, activations) -- so
each process's allocation is that GPU's footprint; only the timing would be distorted by the
sharing, and none is reported.  Per rank and mode (LLEP, then standard EP on a fresh context):

    peak = torch.cuda.max_memory_allocated() (after a reset at the start of the mode)
           + ctx.device_bytes()          (the library's own cudaMalloc: arena + scratch + A)

over two layer calls.  Also printed: the §8(a) memory-model estimate from the plan's g_a[d] and
|S_d| (resident M·6DH + imported |S_d|·6DH + home x,out + R_d·(2D+2H+2D+8)), and whether the LLEP
and EP outputs are bitwise equal.  One JSON line per (config, P, scenario).

    python tools/mem_sweep.py --config g120 --world 8 --scenarios 95:1,95:4,95:16,50:1,30:1,0:0
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def worker(rank, P, cfg, pct, nhot, q, modes=("llep", "ep")):
    import torch
    import torch.distributed as dist
    import layer_case as LC
    from synth import workload as W
    from paper_2601_17111_b200 import llep as L

    dist.init_process_group("gloo", rank=rank, world_size=P)
    torch.cuda.set_device(0)
    sh0 = W.CONFIGS[cfg]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
    x, ids, gates, w13, w2, _, _ = LC.rank_inputs(sh, rank, None if pct == 0 else pct, nhot, 21, "cuda:0")
    res = {}
    outs = {}
    for mode in modes:
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, P, rank, 0, sh.tokens_per_rank)
        for _ in range(2):
            out = ctx(x, ids, gates, w13, w2, ep=(mode == "ep"))
        torch.cuda.synchronize()
        plan = L.parse_plan(bytes(ctx.prepare(ids, ep=(mode == "ep"))[0].cpu().numpy().tobytes()))
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated() + ctx.device_bytes()
        outs[mode] = out
        res[mode] = dict(peak_bytes=int(peak), lib_bytes=int(ctx.device_bytes()),
                         rows=int(plan.assigned[rank]),
                         imported=int(sum(1 for (e, s, d) in plan.transfers if d == rank)),
                         transfers=len(plan.transfers), fallback=bool(plan.fallback))
        dist.barrier()
        ctx.close()
        torch.cuda.synchronize()
    res["same"] = bool(torch.equal(outs["llep"], outs["ep"])) if len(outs) == 2 else None
    gathered = [None] * P
    dist.all_gather_object(gathered, res)
    if rank == 0:
        q.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def model_bytes(sh, M, rows, imported):
    D, H = sh.d_model, sh.d_ff
    return (M + imported) * 6 * D * H + 2 * sh.tokens_per_rank * 2 * D + rows * (2 * D + 2 * H + 2 * D + 8)


def main():
    import torch.multiprocessing as mp
    from synth import workload as W
    from paper_2601_17111_b200 import llep as L
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="g120")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--scenarios", default="95:1,0:0")
    ap.add_argument("--port", type=int, default=29710)
    ap.add_argument("--modes", default="llep,ep",
                    help="llep only for shapes whose EP arenas of all P ranks exceed one GPU (Q3 at P=8)")
    args = ap.parse_args()
    P = args.world
    sh0 = W.CONFIGS[args.config]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
    M = sh.n_experts // P
    ctxm = mp.get_context("spawn")
    for i, sc in enumerate(args.scenarios.split(",")):
        pct, nhot = (int(v) for v in sc.split(":"))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(args.port + i))
        q = ctxm.SimpleQueue()
        modes = tuple(args.modes.split(","))
        mp.spawn(worker, args=(P, args.config, pct, nhot, q, modes), nprocs=P, join=True)
        ranks = q.get()
        line = {"config": args.config, "world": P,
                "scenario": "balanced" if pct == 0 else f"{pct}pct_into_{nhot}", "tokens_per_rank": sh.tokens_per_rank}
        for mode in modes:
            pk = [r[mode]["peak_bytes"] for r in ranks]
            crit = max(range(P), key=lambda p: pk[p])
            line[mode] = {"peak_gb_per_gpu": max(pk) / 1e9, "peak_gb_by_rank": [round(v / 1e9, 3) for v in pk],
                          "critical_rank": crit, "rows_critical": ranks[crit][mode]["rows"],
                          "max_rows": max(r[mode]["rows"] for r in ranks),
                          "lib_gb_critical": ranks[crit][mode]["lib_bytes"] / 1e9,
                          "model_gb_critical": model_bytes(sh, M, ranks[crit][mode]["rows"],
                                                           ranks[crit][mode]["imported"]) / 1e9,
                          "transfers": ranks[0][mode]["transfers"], "fallback": ranks[0][mode]["fallback"]}
        if "ep" not in modes:   # EP not run: its critical rank's memory-model estimate from the EP plan
            ep = L.plan_host((W.slot_counts(sh.n_experts, sh.tokens_per_rank * sh.top_k,
                                            None if pct == 0 else pct, nhot) * P).tolist(), P, ep=True)
            line["ep"] = {"peak_gb_per_gpu": None, "max_rows": max(ep.assigned),
                          "model_gb_critical": model_bytes(sh, M, max(ep.assigned), 0) / 1e9,
                          "note": "not run: P symmetric EP arenas do not fit one GPU"}
        else:
            line["ep_over_llep_peak"] = line["ep"]["peak_gb_per_gpu"] / line["llep"]["peak_gb_per_gpu"]
            line["llep_equals_ep_bitwise"] = all(r["same"] for r in ranks)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
