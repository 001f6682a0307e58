"""Spawn P ranks (processes) that share one GPU and run the LLEP and EP layer through the C ABI.

    python mp_layer_worker.py P CFG HOT_PCT N_HOT OUTDIR        (CFG: a synth.CONFIGS name or shape:N,K,D,H,B)

The ranks bootstrap a gloo process group on 127.0.0.1 (plumbing only: it carries the 64-byte CUDA
IPC handles); all data moves through the library's peer-mapped arenas and device barriers.
Each rank writes OUTDIR/rank{p}.npz with its LLEP output, EP output (the first SAMPLE rows if given, or
the rows listed under key r{p} of the .npz file named by LLEP_TEST_ROWS), the plan blob, whether the
whole LLEP and EP outputs are bitwise equal, and the index work of both calls (load matrix, stable
local ranks, per-slot (device, row) destinations and this rank's group table) for bit-exact comparison
with the oracle O2."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def dump_index_work(L, ctx, sh, P, key):
    """The index work of the last prepare + forward (rows a1-a5): C [P, N], r_j [B*K], (dev, row) [B*K, 2]
    and this rank's group table [G, 8] = (expert, weight slot, row_base, n_rows, mblk_start, 0, 0, 0)."""
    import torch
    BK = sh.tokens_per_rank * sh.top_k
    G = int(ctx.last_req.my_groups)
    return {f"{key}_lm": ctx.debug(L.DBG_LOAD_MATRIX, P * sh.n_experts, torch.int32).cpu().numpy().reshape(P, -1),
            f"{key}_lr": ctx.debug(L.DBG_LOCAL_RANK, BK, torch.int32).cpu().numpy(),
            f"{key}_dst": ctx.debug(L.DBG_SLOT_DST, 2 * BK, torch.int32).cpu().numpy().reshape(-1, 2),
            f"{key}_groups": ctx.debug(L.DBG_GROUPS, 8 * G, torch.int32).cpu().numpy().reshape(G, 8)}


def worker(rank, P, cfg, pct, nhot, outdir, sample):
    import torch
    import torch.distributed as dist
    import layer_case as LC
    from synth import workload as W
    from paper_2601_17111_b200 import llep as L

    dist.init_process_group("gloo", rank=rank, world_size=P)
    dev = int(os.environ.get("LLEP_TEST_DEVICE", "0"))
    torch.cuda.set_device(dev)
    sh0 = LC.config_shape(cfg)
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
    x, ids, gates, w13, w2, _, _ = LC.rank_inputs(sh, rank, None if pct == 0 else pct, nhot, 21, f"cuda:{dev}")
    alpha, m, lam = (float(v) for v in os.environ.get("LLEP_TEST_PARAMS", "1,1024,1.3").split(","))
    m = int(m)
    trace = os.environ.get("LLEP_TEST_TRACE")
    if trace:   # row f4: replay every record of a SPEC-format trace on one context, LLEP and EP
        recs = W.load_trace(trace, sh.n_experts, P)
        bmax = max(int(C[p].sum()) // sh.top_k for C in recs for p in range(P))
        ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, P, rank, dev, bmax)
        xa = W.tokens_torch(bmax, sh.d_model, rank, f"cuda:{dev}", 21)
        res = {}
        for i, C in enumerate(recs):
            ids_np = W.routing_from_counts(C[rank], sh.top_k, rank, 21 + i)
            B = ids_np.shape[0]
            g_np = W.gate_weights(B, sh.top_k, rank, 21 + i)
            ids_t, g_t = torch.from_numpy(ids_np).to(f"cuda:{dev}"), torch.from_numpy(g_np).to(f"cuda:{dev}")
            o1 = ctx(xa[:B], ids_t, g_t, w13, w2, alpha, m, lam)
            o2 = ctx(xa[:B], ids_t, g_t, w13, w2, ep=True)
            torch.cuda.synchronize()
            res[f"r{i}_llep"] = o1.float().cpu().numpy()
            res[f"r{i}_same"] = np.array(bool(torch.equal(o1, o2)))
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), n_records=np.array(len(recs)), **res)
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()
        return
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, P, rank, dev, sh.tokens_per_rank)
    if os.environ.get("LLEP_TEST_ORDER"):   # the token order of a3/a5 (default chunk-aligned)
        ctx.set_token_order(os.environ["LLEP_TEST_ORDER"])
    out_llep = ctx(x, ids, gates, w13, w2, alpha, m, lam)
    plan = ctx.prepare(ids, alpha, m, lam)[0]          # plan of the LLEP call (deterministic)
    plan_np = plan.cpu().numpy()
    out_llep2 = ctx.forward(x, ids, gates, w13, w2, plan)   # second iteration on the same arena
    index_work = dump_index_work(L, ctx, sh, P, "llep")
    out_ep = ctx(x, ids, gates, w13, w2, ep=True)
    index_work.update(dump_index_work(L, ctx, sh, P, "ep"))
    torch.cuda.synchronize()
    assert torch.equal(out_llep, out_llep2), "iteration-to-iteration mismatch"
    n = sample if sample > 0 else out_llep.shape[0]
    rows_file = os.environ.get("LLEP_TEST_ROWS")
    sel = slice(0, n)
    if rows_file:
        sel = torch.from_numpy(np.load(rows_file)[f"r{rank}"].astype(np.int64)).to(out_llep.device)
    extra = dict(index_work)
    if os.environ.get("LLEP_TEST_BWD") == "1":
        ctx.enable_backward()
        dout = W.tokens_torch(sh.tokens_per_rank, sh.d_model, rank + 1000, f"cuda:{dev}", 21)
        plan_b, _ = ctx.prepare(ids, alpha, m, lam)
        dx, dg, dw13, dw2 = ctx.backward(x, ids, gates, dout, w13, w2, plan_b)
        torch.cuda.synchronize()
        # training path: forward that saves [g | u], backward from the saved values == recompute
        _, gu = ctx.forward_train(x, ids, gates, w13, w2, plan_b)
        saved = ctx.backward(x, ids, gates, dout, w13, w2, plan_b, gu=gu)
        torch.cuda.synchronize()
        for a_, b_ in zip(saved, (dx, dg, dw13, dw2)):
            assert torch.equal(a_, b_), "saved-preactivation backward differs from the recompute"
        extra.update(dx=dx[sel].float().cpu().numpy(), dgates=dg[sel].cpu().numpy(), dw13=dw13.cpu().numpy(),
                     dw2=dw2.cpu().numpy())
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), llep=out_llep[sel].float().cpu().numpy(),
             ep=out_ep[sel].float().cpu().numpy(), plan=plan_np,
             same=np.array(bool(torch.equal(out_llep, out_ep))), **extra)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    P, cfg, pct, nhot, outdir = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    sample = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    mp.spawn(worker, args=(P, cfg, pct, nhot, outdir, sample), nprocs=P, join=True)
