"""Independent cross-check of the NVLink dispatch: P ranks, one GPU each, NCCL process group.
Each rank runs llep_prepare + llep_moe_forward, reads back its receive rows (LLEP_DBG_RECV_X) and rebuilds
the same rows with torch.distributed.all_to_all_single: every source sends, for each slot, its token row
and the destination row index (from its own slot_dst of the same plan); the destination scatters the
received rows to those indices.  Writes OUTDIR/xcheck{p}.npz with the number of rows compared and
whether they are bitwise equal.

    torchrun --nproc-per-node P mp_nccl_xcheck_worker.py OUTDIR CFG HOT NHOT
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    # the check reads the receive buffer: the dispatch must copy every row, including the local rows
    # GEMM1 would gather straight from x under the opt-in LLEP_GATHER=1 (a6 local rows)
    os.environ.pop("LLEP_GATHER", None)
    import torch
    import torch.distributed as dist
    import layer_case as LC
    from synth import workload as W
    from paper_2601_17111_b200 import llep as L
    outdir, cfg, hot, nhot = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device(f"cuda:{rank}")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    sh0 = W.CONFIGS[cfg]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
    x, ids, gates, w13, w2, ids_np, _ = LC.rank_inputs(sh, rank, None if hot == 0 else hot, nhot, 21, dev)
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, P, rank, rank, sh.tokens_per_rank,
                    group=dist.group.WORLD)
    ctx(x, ids, gates, w13, w2)
    torch.cuda.synchronize()
    BK = sh.tokens_per_rank * sh.top_k
    dst = ctx.debug(L.DBG_SLOT_DST, 2 * BK, torch.int32).view(-1, 2).long()
    rows_here = int(ctx.last_req.rows_needed)
    recv_x = ctx.debug(L.DBG_RECV_X, rows_here * sh.d_model, torch.bfloat16).view(rows_here, sh.d_model)
    # NCCL all-to-all of the same rows: order this rank's slots by destination device
    tok = torch.arange(BK, device=dev) // sh.top_k
    order = torch.argsort(dst[:, 0], stable=True)
    send_counts = torch.bincount(dst[:, 0], minlength=P)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts)
    sc, rc = send_counts.tolist(), recv_counts.tolist()
    send_rows = x[tok[order]].contiguous()
    send_idx = dst[order, 1].to(torch.int32).contiguous()
    got_rows = torch.empty((sum(rc), sh.d_model), dtype=torch.bfloat16, device=dev)
    got_idx = torch.empty(sum(rc), dtype=torch.int32, device=dev)
    dist.all_to_all_single(got_rows, send_rows, rc, sc)
    dist.all_to_all_single(got_idx, send_idx, rc, sc)
    ref = torch.zeros_like(recv_x)
    ref[got_idx.long()] = got_rows
    mine = recv_x[got_idx.long()]
    same = bool(torch.equal(mine, got_rows))
    np.savez(os.path.join(outdir, f"xcheck{rank}.npz"), rows=np.array(sum(rc)), same=np.array(same),
             sent=np.array(sc), received=np.array(rc))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
