"""Capture-safe layer call (llep_moe_layer): prepare + forward with no host synchronisation, captured
in a CUDA graph and replayed with new routings; every output bit-identical to the two-call path."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import layer_case as LC  # noqa: E402
import mp_graph_worker as GW  # noqa: E402
from synth import workload as W  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_17111_b200 import llep
    return llep


@pytest.mark.parametrize("cfg,B", [("tiny", 1024), ("g20", 4096), ("q3", 4096)])
def test_layer_graph_replay_p1(L, cfg, B):
    base = W.CONFIGS[cfg]
    sh = W.LayerShape(base.n_experts, base.top_k, base.d_model, base.d_ff, B, 1)
    x = W.tokens_torch(B, sh.d_model, 0, "cuda", 21)
    w13, w2 = W.expert_weights_torch(range(sh.n_experts), sh.d_model, sh.d_ff, "cuda", 21)
    R = [(torch.from_numpy(i).cuda(), torch.from_numpy(g).cuda()) for i, g in GW.routings(sh, 0)]
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, 1, 0, 0, B)
    ref = [ctx(x, ids, g, w13, w2).clone() for ids, g in R]
    for (ids, g), r in zip(R, ref):   # direct (uncaptured) layer calls
        assert torch.equal(ctx.layer(x, ids, g, w13, w2), r)
    ids_s, g_s = R[0][0].clone(), R[0][1].clone()
    plan_s = torch.empty(L.plan_bytes(sh.n_experts, 1), dtype=torch.uint8, device="cuda")
    out_s = torch.empty((B, sh.d_model), dtype=torch.bfloat16, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        ctx.layer(x, ids_s, g_s, w13, w2, plan_out=plan_s, out=out_s)
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ctx.layer(x, ids_s, g_s, w13, w2, plan_out=plan_s, out=out_s)
    for i in (1, 3, 0, 2, 1):
        ids_s.copy_(R[i][0])
        g_s.copy_(R[i][1])
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(out_s, ref[i]), i
    ctx.check()
    # and against the float64 oracle for the last replayed routing (first rows)
    ids_np, g_np = GW.routings(sh, 0)[1]
    rows = np.arange(min(B, 128))
    refo = LC.oracle_rank_output(sh, 0, ids_np, g_np, 21, rows=rows)
    mr, l2 = LC.errors(out_s[: len(rows)].float().cpu().numpy().astype(np.float64), refo)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (mr, l2)
    del graph
    ctx.close()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_layer_graph_replay_processes(L, tmp_path, P):
    """P processes on one GPU: direct layer calls (LLEP and EP) and graph replays with changing routings
    == the two-call path bit for bit; an EP plan larger than a fresh arena is caught on the device
    (LLEP_ERR_PLAN at the next check) and the context recovers.  At P=8 the hot expert's 7 replicas take
    three levels of the GPU-issued broadcast tree (native -> 1, 2, 4; 1 -> 3, 5; 2 -> 6; 3 -> 7)."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29650 + P))
    cmd = [sys.executable, os.path.join(HERE, "mp_graph_worker.py"), str(P), "tiny", str(tmp_path)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for p in range(P):
        res = np.load(os.path.join(tmp_path, f"rank{p}.npz"))
        assert res["direct_same"].all(), (p, res["direct_same"])
        assert res["replay_same"].all(), (p, res["replay_same"])
        assert int(res["overflow_code"]) == 2, (p, int(res["overflow_code"]))


def test_layer_small_and_empty_batches_p1(L):
    """The capture-safe call on B = 0, 1, 7 and a ragged 1000 tokens == the two-call path bit for bit."""
    sh = W.LayerShape(8, 2, 256, 512, 1024, 1)
    x = W.tokens_torch(1024, 256, 0, "cuda", 5)
    ids = torch.from_numpy(W.routing_ids(sh, 0, 95, 1, 5)).cuda()
    g = torch.from_numpy(W.gate_weights(1024, 2, 0, 5)).cuda()
    w13, w2 = W.expert_weights_torch(range(8), 256, 512, "cuda", 5)
    ctx = L.Context(8, 2, 256, 512, 1, 0, 0, 1024)
    for B in (0, 1, 7, 1000):
        xs, ii, gg = x[:B].contiguous(), ids[:B].contiguous(), g[:B].contiguous()
        a = ctx(xs, ii, gg, w13, w2).clone()
        b = ctx.layer(xs, ii, gg, w13, w2)
        torch.cuda.synchronize()
        assert torch.equal(a, b), B
    ctx.check()
    ctx.close()


@pytest.mark.parametrize("P,cfg,n,seed,port", [(2, "tiny", 24, 101, 29671), (4, "tiny", 24, 202, 29672),
                                               (8, "tiny", 16, 303, 29673), (4, "g20", 6, 404, 29674),
                                               (8, "dsv3", 3, 505, 29675)])
def test_layer_call_fuzz_processes(L, tmp_path, P, cfg, n, seed, port):
    """Random skews and planner parameters (spills, force-assigns, λ fallbacks, EP): the capture-safe
    call == the two-call path bit for bit on every rank, and the cases exercise every plan kind."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    cmd = [sys.executable, os.path.join(HERE, "mp_layer_fuzz_worker.py"), str(P), cfg, str(n), str(seed), str(tmp_path)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"fuzz{p}.npz")) for p in range(P)]
    for p in range(P):
        assert res[p]["same"].all(), (p, np.nonzero(~res[p]["same"])[0], res[p]["info"][~res[p]["same"]])
    info = res[0]["info"]
    assert (info[:, 7] > 0).any()                        # some plans spill (weight transfers)
    if n >= 16:
        assert (info[:, 9] > 0).any()                    # and some fall back to EP (λ test)
