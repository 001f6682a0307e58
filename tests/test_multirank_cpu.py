"""The N>1 host path on CPU with world-size-2 (and 4) gloo process groups -- no GPU: per-rank inputs,
the count exchange + host planner giving one plan on every rank (== the oracle O1), the max-over-ranks
helpers, bench.py's NVLink byte accounting (pinned by O2's per-slot destinations), and the reference arm
under torchrun (rank 0 alone prints the line)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


@pytest.mark.parametrize("P,cfg,pct,nhot,port", [(2, "tiny", 95, 1, 29711), (2, "g120", 95, 1, 29712),
                                                 (4, "g120", 95, 4, 29713), (2, "tiny", 0, 0, 29714)])
def test_gloo_ranks_agree_on_plan_and_link_bytes(tmp_path, P, cfg, pct, nhot, port):
    from oracle import planner as O1
    from oracle import schedule as O2
    from synth import workload as W
    cmd = [sys.executable, os.path.join(HERE, "mp_cpu_worker.py"), str(P), cfg, str(pct), str(nhot),
           str(tmp_path), str(port)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"cpu{p}.npz")) for p in range(P)]
    sh0 = W.CONFIGS[cfg]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
    ids_all = [W.routing_ids(sh, p, None if pct == 0 else pct, nhot, 21) for p in range(P)]
    C = O2.load_matrix(ids_all, sh.n_experts)
    ref = O1.plan(C.sum(0).tolist(), P)
    for p in range(P):
        assert np.array_equal(res[p]["ids"], ids_all[p])            # rank-seeded inputs, per rank
        assert np.array_equal(res[p]["C"], C)                         # the exchanged load matrix
        assert bool(res[p]["plans_equal"])                            # one plan on every rank
        assert float(res[p]["max_over_ranks"]) == 10 * (P - 1) + 1
        assert int(res[p]["max_tokens"]) == 1000 + P - 1
        assert int(res[p]["n_transfers"]) == len(ref.transfers)
    # NVLink byte accounting of bench.py vs the oracle's per-slot destinations: every (token, slot)
    # routed to a device other than its home rank crosses once each way; every replica gets one copy
    D, H = sh.d_model, sh.d_ff
    remote = 0
    for p in range(P):
        dev, _row = O2.slot_destinations(ref, C, ids_all[p], p, aligned=True)   # the default order (R11')
        remote += int((dev != p).sum())
    assert int(res[0]["disp"]) == remote * (2 * D + 8)
    assert int(res[0]["comb"]) == remote * 2 * D
    assert int(res[0]["wts"]) == len(ref.transfers) * 6 * D * H
    if pct is None or pct == 0:
        assert remote == sum(int(((ids_all[p] // sh.experts_per_rank) != p).sum()) for p in range(P))


def test_reference_arm_under_torchrun_world2():
    """bench.py --impl reference --gpus 2 under torchrun: rank 0 alone runs the oracle and prints ONE
    contract line; rank 1 exits 0 without work."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29721", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "3", "--config", "tiny"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["value"] > 0 and d["unit"] == "tokens/s"
