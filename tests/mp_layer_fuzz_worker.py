"""Fuzz of the capture-safe layer call against the two-call path at P > 1 (processes sharing one GPU):
random skews (1/4/16 hot experts, sampled or exact counts, balanced), random planner parameters (α, m, λ)
so that spills, force-assigns and λ fallbacks all occur, LLEP and EP, and ragged batches (each rank its own
token count, some ranks empty); per case the direct llep_moe_layer
output must equal the two-call output bit for bit and leave no device error.

    python mp_layer_fuzz_worker.py P CFG N_CASES SEED OUTDIR    -> OUTDIR/fuzz{p}.npz"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def worker(rank, P, cfg, n_cases, seed, outdir):
    import torch
    import torch.distributed as dist
    from synth import workload as W
    from paper_2601_17111_b200 import llep as L
    dist.init_process_group("gloo", rank=rank, world_size=P)
    torch.cuda.set_device(0)
    d = "cuda:0"
    sh0 = W.CONFIGS[cfg]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
    B, M = sh.tokens_per_rank, sh.experts_per_rank
    x = W.tokens_torch(B, sh.d_model, rank, d, seed)
    w13, w2 = W.expert_weights_torch(range(rank * M, (rank + 1) * M), sh.d_model, sh.d_ff, d, seed)
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, P, rank, 0, B, group=dist.group.WORLD)
    rng = np.random.default_rng(seed)          # same draws on every rank: same case parameters
    same, info = [], []
    for i in range(n_cases):
        pct = int(rng.choice([0, 30, 50, 80, 95]))
        nhot = min(int(rng.choice([1, 4, 16])), sh.n_experts - 1)
        sampled = bool(rng.integers(0, 2))
        shift = int(rng.integers(0, sh.n_experts))
        alpha = float(rng.choice([1.0, 1.1, 1.5]))
        m = int(rng.choice([1, 16, 256, 1024]))
        lam = float(rng.choice([1.0, 1.3, 3.0]))
        ep = bool(rng.integers(0, 4) == 0)
        ragged = bool(rng.integers(0, 3) == 0)   # every third case: a different batch per rank, some empty
        ids = W.routing_ids(sh, rank, None if pct == 0 else pct, nhot, seed + 7 * i, sampled=sampled)
        ids = torch.from_numpy(((ids + shift) % sh.n_experts).astype(np.int32)).to(d)
        g = torch.from_numpy(W.gate_weights(B, sh.top_k, rank, seed + i)).to(d)
        xb = x
        if ragged:
            r_rng = np.random.default_rng([seed, i, rank])
            Br = int(r_rng.choice([0, 1, 7, B // 3, B]))
            xb, ids, g = x[:Br].contiguous(), ids[:Br].contiguous(), g[:Br].contiguous()
        a = ctx(xb, ids, g, w13, w2, alpha, m, lam, ep=ep).clone()
        req = ctx.last_req
        b = ctx.layer(xb, ids, g, w13, w2, alpha, m, lam, ep=ep)
        torch.cuda.synchronize()
        ctx.check()
        same.append(bool(torch.equal(a, b)))
        info.append((pct, nhot, int(sampled), alpha, m, lam, int(ep), int(req.n_transfers), int(req.force_count),
                     int(req.fallback_ep)))
    np.savez(os.path.join(outdir, f"fuzz{rank}.npz"), same=np.array(same), info=np.array(info, dtype=np.float64))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    P, cfg, n, seed, outdir = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    mp.spawn(worker, args=(P, cfg, n, seed, outdir), nprocs=P, join=True)
