"""P ranks (processes sharing one GPU, CUDA-IPC arenas) run the capture-safe llep_moe_layer: direct calls
and CUDA-graph replays with new routings copied into the captured input buffers, each compared bit for bit
with the two-call path (llep_prepare + llep_moe_forward) on the same inputs; plus the device-side arena
overflow check.

    python mp_graph_worker.py P CFG OUTDIR

Writes OUTDIR/rank{p}.npz: direct_same[r], replay_same[r] (bool per routing r), overflow_code."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def routings(sh, rank, seed=21):
    """(ids, gates) per routing: 95 %/1 with the hot expert on rank 0, the same shifted to rank 1's
    natives, balanced, 50 %/4 -- so every replay has a different plan."""
    from synth import workload as W
    B, K, N, M = sh.tokens_per_rank, sh.top_k, sh.n_experts, sh.experts_per_rank
    hot = W.routing_ids(sh, rank, 95, 1, seed)
    out = [hot, ((hot + M) % N).astype(np.int32), W.routing_ids(sh, rank, None, 0, seed),
           W.routing_ids(sh, rank, 50, 4, seed)]
    return [(ids, W.gate_weights(B, K, rank, seed + i)) for i, ids in enumerate(out)]


def worker(rank, P, cfg, outdir):
    import torch
    import torch.distributed as dist
    from synth import workload as W
    from paper_2601_17111_b200 import llep as L

    dist.init_process_group("gloo", rank=rank, world_size=P)
    dev = int(os.environ.get("LLEP_TEST_DEVICE", "0"))
    torch.cuda.set_device(dev)
    d = f"cuda:{dev}"
    sh0 = W.CONFIGS[cfg]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
    B, M = sh.tokens_per_rank, sh.experts_per_rank
    x = W.tokens_torch(B, sh.d_model, rank, d, 21)
    w13, w2 = W.expert_weights_torch(range(rank * M, (rank + 1) * M), sh.d_model, sh.d_ff, d, 21)
    R = [(torch.from_numpy(i).to(d), torch.from_numpy(g).to(d)) for i, g in routings(sh, rank)]

    # arena overflow on the device: EP of the 95 %/1 routing needs more rows than a fresh arena holds
    small = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, P, rank, dev, B, group=dist.group.WORLD)
    small.layer(x, R[0][0], R[0][1], w13, w2, ep=True)
    code = 0
    try:
        small.check()
    except L.LLEPError as e:
        code = e.code
    small.layer(x, R[2][0], R[2][1], w13, w2)   # a balanced plan fits: the context recovers
    small.check()
    small.close()

    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, P, rank, dev, B, group=dist.group.WORLD)
    ref = []
    for ids, g in R:   # two-call path; prepare() grows the arena (symmetrically) to every plan's needs
        ref.append(ctx(x, ids, g, w13, w2).clone())
        ref.append(ctx(x, ids, g, w13, w2, ep=True).clone())
    torch.cuda.synchronize()
    direct = []
    for i, (ids, g) in enumerate(R):
        o = ctx.layer(x, ids, g, w13, w2)
        oe = ctx.layer(x, ids, g, w13, w2, ep=True)
        torch.cuda.synchronize()
        direct.append(bool(torch.equal(o, ref[2 * i])) and bool(torch.equal(oe, ref[2 * i + 1])))
    ctx.check()
    # capture one layer call, replay it with every routing copied into the captured buffers
    ids_s, g_s = R[0][0].clone(), R[0][1].clone()
    plan_s = torch.empty(L.plan_bytes(sh.n_experts, P), dtype=torch.uint8, device=d)
    out_s = torch.empty((B, sh.d_model), dtype=torch.bfloat16, device=d)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):   # warm-up on a side stream, as torch.cuda.graph expects
        ctx.layer(x, ids_s, g_s, w13, w2, plan_out=plan_s, out=out_s)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    dist.barrier()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ctx.layer(x, ids_s, g_s, w13, w2, plan_out=plan_s, out=out_s)
    torch.cuda.synchronize()
    dist.barrier()
    replay = []
    for i in (1, 0, 3, 2, 1):
        ids_s.copy_(R[i][0])
        g_s.copy_(R[i][1])
        graph.replay()
        torch.cuda.synchronize()
        replay.append(bool(torch.equal(out_s, ref[2 * i])))
    ctx.check()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), direct_same=np.array(direct), replay_same=np.array(replay),
             overflow_code=np.array(code))
    dist.barrier()
    del graph
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    P, cfg, outdir = int(sys.argv[1]), sys.argv[2], sys.argv[3]
    mp.spawn(worker, args=(P, cfg, outdir), nprocs=P, join=True)
