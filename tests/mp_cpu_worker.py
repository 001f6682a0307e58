"""World-size-2 (or more) gloo worker for the CPU multi-rank tests: the host side of the N>1 path.

Each rank draws its own routing (synth, rank-seeded), exchanges its per-expert counts with the other
ranks (all_gather, the host analogue of the a2 push), plans with the C-ABI host planner, and reports its
plan blob, the per-rank max helpers of llep.py / bench.py and bench.py's NVLink byte accounting, so the
parent test can check that every rank agrees and matches the oracle."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


def worker(rank, P, cfg, pct, nhot, outdir, port):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    import bench
    from synth import workload as W
    from paper_2601_17111_b200 import llep as L
    sh0 = W.CONFIGS[cfg]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
    ids = W.routing_ids(sh, rank, pct, nhot, 21)
    cnt = torch.from_numpy(np.bincount(ids.ravel(), minlength=sh.n_experts).astype(np.int64))
    allc = [torch.zeros_like(cnt) for _ in range(P)]
    dist.all_gather(allc, cnt)
    C = torch.stack(allc).numpy()
    plan = L.plan_host(C.sum(0).tolist(), P, 1.0, 1024, 1.3)
    links = bench.link_bytes(plan, C, sh.d_model, sh.d_ff)
    mx = bench.max_over_ranks(float(rank * 10 + 1), P)
    mt = L._max_over_group(1000 + rank, None)
    chunks = [list(map(list, A)) for A in plan.chunks]
    allplans = [None] * P
    dist.all_gather_object(allplans, chunks)
    np.savez(os.path.join(outdir, f"cpu{rank}.npz"), C=C, ids=ids, max_over_ranks=mx, max_tokens=mt,
             plans_equal=np.array(all(p == chunks for p in allplans)),
             disp=links["dispatch"]["total_bytes"], comb=links["combine"]["total_bytes"],
             wts=links["weights"]["total_bytes"], n_transfers=len(plan.transfers))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    P, cfg, pct, nhot, outdir, port = (int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4]),
                                      sys.argv[5], int(sys.argv[6]))
    mp.spawn(worker, args=(P, cfg, None if pct == 0 else pct, nhot, outdir, port), nprocs=P, join=True)
