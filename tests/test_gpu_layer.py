"""End-to-end layer parity on the GPU: CUDA path (C ABI) vs the float64 oracle (O1-O3)."""
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
from synth import workload as W  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_17111_b200 import llep
    return llep


def _to_np(t):
    return t.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("cfg,pct,nhot,ep", [
    ("tiny", 95, 1, False), ("tiny", 95, 1, True), ("tiny", None, 0, False), ("tiny", 50, 4, False),
])
def test_layer_p1_full_parity(L, cfg, pct, nhot, ep):
    """P=1 (every expert native): whole output vs O3, plus the internal a1/a3 steps vs O2."""
    from oracle import schedule as O2
    base = W.CONFIGS[cfg]
    sh = W.LayerShape(base.n_experts, base.top_k, base.d_model, base.d_ff, base.tokens_per_rank, 1)
    seed = 11
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, pct, nhot, seed, "cuda")
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, 1, 0, 0, sh.tokens_per_rank)
    out = ctx(x, ids, gates, w13, w2, ep=ep)
    torch.cuda.synchronize()
    ref = LC.oracle_rank_output(sh, 0, ids_np, g_np, seed)
    mr, l2 = LC.errors(_to_np(out), ref)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (mr, l2)
    # a1: load matrix; a3: stable local ranks (bit-exact)
    lm = ctx.debug(L.DBG_LOAD_MATRIX, sh.n_experts, torch.int32).cpu().numpy()
    assert np.array_equal(lm, O2.local_counts(ids_np, sh.n_experts))
    lr = ctx.debug(L.DBG_LOCAL_RANK, ids_np.size, torch.int32).cpu().numpy()
    assert np.array_equal(lr, O2.local_rank_in_expert(ids_np))
    ctx.close()


def test_layer_empty_and_small_batches(L):
    """B = 0, 1 and a ragged tail: valid outputs, no errors."""
    sh = W.LayerShape(8, 2, 256, 512, 1024, 1)
    ctx = L.Context(8, 2, 256, 512, 1, 0, 0, 1024)
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, 95, 1, 5, "cuda")
    for B in (0, 1, 7, 1000):
        out = ctx(x[:B].contiguous(), ids[:B].contiguous(), gates[:B].contiguous(), w13, w2)
        torch.cuda.synchronize()
        if B:
            ref = LC.oracle_rank_output(sh, 0, ids_np[:B], g_np[:B], 5)
            mr, l2 = LC.errors(_to_np(out), ref)
            assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (B, mr, l2)
    ctx.close()


def test_routing_error_reported(L):
    ctx = L.Context(8, 2, 256, 512, 1, 0, 0, 64)
    ids = torch.zeros((16, 2), dtype=torch.int32, device="cuda")
    ids[3, 1] = 9
    with pytest.raises(L.LLEPError) as ei:
        ctx.prepare(ids)
    assert ei.value.code == 3
    ids[3, 1] = 1
    ctx.prepare(ids)  # recovers
    ctx.close()


def test_multiprocess_p2_p4_one_gpu(L, tmp_path):
    """P ranks as P processes sharing cuda:0, arenas mapped through CUDA IPC: every output vs O3,
    LLEP vs EP, plan identical on every rank and == the oracle plan."""
    for P, cfg, pct, nhot in [(2, "tiny", 95, 1), (4, "tiny", 80, 1)]:
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29500 + P))
        cmd = [sys.executable, os.path.join(HERE, "mp_layer_worker.py"), str(P), cfg, str(pct), str(nhot),
               str(tmp_path)]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        res = [np.load(os.path.join(tmp_path, f"rank{p}.npz")) for p in range(P)]
        sh0 = W.CONFIGS[cfg]
        sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
        from oracle import planner as O1
        from oracle import schedule as O2
        ids_all = [W.routing_ids(sh, p, pct, nhot, 21) for p in range(P)]
        C = O2.load_matrix(ids_all, sh.n_experts)
        ref_plan = O1.plan(C.sum(0).tolist(), P)
        plans = [bytes(r_["plan"].tobytes()) for r_ in res]
        assert all(p == plans[0] for p in plans)
        dp = L.parse_plan(plans[0])
        assert [list(A) for A in dp.chunks] == [list(A) for A in ref_plan.chunks]
        assert len(ref_plan.transfers) > 0  # the spill path is exercised
        LC.check_index_work(res, "llep", ref_plan, ids_all, sh.n_experts)
        LC.check_index_work(res, "ep", O1.ep_plan(C.sum(0).tolist(), P, 1.0, fallback=False), ids_all,
                            sh.n_experts)
        w = LC.OracleWeights(sh.d_model, sh.d_ff, 21)
        for p in range(P):
            ref = LC.oracle_rank_output(sh, p, ids_all[p], W.gate_weights(sh.tokens_per_rank, sh.top_k, p, 21), 21,
                                        weights=w)
            for key in ("llep", "ep"):
                mr, l2 = LC.errors(res[p][key].astype(np.float64), ref)
                assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (P, p, key, mr, l2)
            # same kernels, fixed K-loop and slot order -> LLEP == EP bitwise (reading R28)
            assert np.array_equal(res[p]["llep"], res[p]["ep"]) and bool(res[p]["same"])


@pytest.mark.parametrize("P,pct,nhot,params", [
    (4, 30, 1, (1.0, 600, 1.3)),      # 2 LLAS force-assigns: one device ends above the capacity
    (4, 60, 2, (1.25, 1500, 1.3)),    # force-assign with α > 1
    (2, 95, 1, (2.0, 16, 1.0)),       # λ = 1 (never falls back), small m
])
def test_multiprocess_force_assign_and_params(L, tmp_path, P, pct, nhot, params):
    """Plans with force-assigns and non-default α/m/λ through the whole layer."""
    from oracle import planner as O1
    from oracle import schedule as O2
    alpha, m, lam = params
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29700 + P + pct),
               LLEP_TEST_PARAMS=f"{alpha},{m},{lam}")
    cmd = [sys.executable, os.path.join(HERE, "mp_layer_worker.py"), str(P), "tiny", str(pct), str(nhot),
           str(tmp_path)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"rank{p}.npz")) for p in range(P)]
    sh0 = W.CONFIGS["tiny"]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
    ids_all = [W.routing_ids(sh, p, pct, nhot, 21) for p in range(P)]
    C = O2.load_matrix(ids_all, sh.n_experts)
    ref_plan = O1.plan(C.sum(0).tolist(), P, alpha, m, lam)
    dp = L.parse_plan(bytes(res[0]["plan"].tobytes()))
    assert [list(A) for A in dp.chunks] == [list(A) for A in ref_plan.chunks]
    assert dp.force_count == ref_plan.force_count
    if (P, pct) != (2, 95):
        assert ref_plan.force_count > 0
    LC.check_index_work(res, "llep", ref_plan, ids_all, sh.n_experts)
    w = LC.OracleWeights(sh.d_model, sh.d_ff, 21)
    for p in range(P):
        ref = LC.oracle_rank_output(sh, p, ids_all[p], W.gate_weights(sh.tokens_per_rank, sh.top_k, p, 21), 21,
                                    weights=w)
        mr, l2 = LC.errors(res[p]["llep"].astype(np.float64), ref)
        assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (p, mr, l2)
        assert bool(res[p]["same"])


def test_q3_p1_sampled_parity(L):
    """Qwen3-30B-A3B-shaped layer (128 experts, top-8, D=2048, H=768, 64K tokens) at P=1."""
    sh0 = W.CONFIGS["q3"]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, 1)
    seed = 41
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, 95, 1, seed, "cuda")
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, 1, 0, 0, sh.tokens_per_rank)
    out = ctx(x, ids, gates, w13, w2)
    torch.cuda.synchronize()
    ok = np.nonzero((ids_np < 12).all(1))[0]
    rows = np.unique(np.concatenate([ok[:40], ok[-24:]]))
    ref = LC.oracle_rank_output(sh, 0, ids_np, g_np, seed, rows=rows)
    mr, l2 = LC.errors(_to_np(out[torch.from_numpy(rows).cuda()]), ref)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (mr, l2)
    ctx.close()


def test_g120_p1_sampled_parity(L):
    """BASELINE config G120 at the N=1 bench launch configuration (P=1, 32K tokens, 95 %/1):
    sampled outputs vs O3 (tokens whose experts all lie in 0..15, plus the first rows)."""
    sh0 = W.CONFIGS["g120"]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, 1)
    seed = 31
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, 95, 1, seed, "cuda")
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, 1, 0, 0, sh.tokens_per_rank)
    out = ctx(x, ids, gates, w13, w2)
    torch.cuda.synchronize()
    ok = np.nonzero((ids_np < 16).all(1))[0]
    rows = np.unique(np.concatenate([ok[:40], ok[-24:], [0]]))
    ref = LC.oracle_rank_output(sh, 0, ids_np, g_np, seed, rows=rows)
    mr, l2 = LC.errors(_to_np(out[torch.from_numpy(rows).cuda()]), ref)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (mr, l2)
    ctx.close()


@pytest.mark.parametrize("cfg,P,pct,nhot,n_tr", [
    ("g120", 8, 95, 1, 7), ("g120", 8, 0, 0, 0),       # the north-star layer at its N=8 configuration
    ("g20", 8, 95, 1, 7),                              # BASELINE configs[1]
    ("g120", 4, 95, 4, 5), ("g120", 2, 95, 16, 8),     # SWEEP rows at EP 4 / EP 2
])
def test_large_layer_processes_one_gpu(L, tmp_path, cfg, P, pct, nhot, n_tr):
    """BASELINE shapes at full size with P ranks (processes sharing cuda:0, CUDA-IPC arenas),
    λ=1.3 α=1 m=1024.  Plan == oracle on every rank (expected weight-transfer count; EP fallback when
    balanced); the index work (load matrix, local ranks, group tables, every slot's (device, row)) of
    the LLEP and EP calls bit-exact vs O2 on every rank; outputs vs O3 on a sample holding the tokens at
    the first and last global index of every plan chunk (every chunk / group boundary of every device)
    plus each rank's first 16 tokens; LLEP == EP bitwise on every full output."""
    from oracle import planner as O1
    from oracle import schedule as O2
    sh0 = W.CONFIGS[cfg]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
    hot = None if pct == 0 else pct
    ids_all = [W.routing_ids(sh, p, hot, nhot, 21) for p in range(P)]
    C = O2.load_matrix(ids_all, sh.n_experts)
    ref_plan = O1.plan(C.sum(0).tolist(), P)
    rows = LC.boundary_tokens(ref_plan, ids_all, sh.n_experts)
    rows_file = os.path.join(tmp_path, "rows.npz")
    np.savez(rows_file, **{f"r{p}": rows[p] for p in range(P)})
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29600 + pct + 7 * P + len(cfg)),
               LLEP_TEST_ROWS=rows_file)
    cmd = [sys.executable, os.path.join(HERE, "mp_layer_worker.py"), str(P), cfg, str(pct), str(nhot),
           str(tmp_path)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"rank{p}.npz")) for p in range(P)]
    plans = [bytes(r_["plan"].tobytes()) for r_ in res]
    assert all(p == plans[0] for p in plans)
    dp = L.parse_plan(plans[0])
    assert [list(A) for A in dp.chunks] == [list(A) for A in ref_plan.chunks]
    assert len(ref_plan.transfers) == n_tr and dp.fallback == (pct == 0)
    LC.check_index_work(res, "llep", ref_plan, ids_all, sh.n_experts)
    LC.check_index_work(res, "ep", O1.ep_plan(C.sum(0).tolist(), P, 1.0, fallback=False), ids_all, sh.n_experts)
    w = LC.OracleWeights(sh.d_model, sh.d_ff, 21)
    n_chunks = sum(len(A) for A in ref_plan.chunks)
    assert sum(len(v) for v in rows.values()) >= min(n_chunks, 16 * P)
    for p in range(P):
        ref = LC.oracle_rank_output(sh, p, ids_all[p], W.gate_weights(sh.tokens_per_rank, sh.top_k, p, 21), 21,
                                    rows=rows[p], weights=w)
        mr, l2 = LC.errors(res[p]["llep"].astype(np.float64), ref)
        assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (p, mr, l2)
        assert bool(res[p]["same"])


def test_g120_p1_full_output_parity(L):
    """BASELINE config G120 at the N=1 bench launch configuration (P=1, 32K tokens, 95 %/1): the WHOLE
    [32768, 2880] output vs the float64 oracle O3 (6.5 TFLOP of float64 on the host; rows of each
    expert processed in chunks), plus the index work (a1, a3, a5) bit-exact vs O2."""
    from oracle import planner as O1
    from oracle import schedule as O2
    sh0 = W.CONFIGS["g120"]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, 1)
    seed = 31
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, 95, 1, seed, "cuda")
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, 1, 0, 0, sh.tokens_per_rank)
    out = ctx(x, ids, gates, w13, w2)
    torch.cuda.synchronize()
    import mp_layer_worker as MW
    res = [MW.dump_index_work(L, ctx, sh, 1, "llep")]
    plan = O1.plan(O2.local_counts(ids_np, sh.n_experts).tolist(), 1)
    LC.check_index_work(res, "llep", plan, [ids_np], sh.n_experts)
    y = _to_np(out)
    ctx.close()
    del out, x, w13, w2
    ref = LC.oracle_rank_output(sh, 0, ids_np, g_np, seed)
    mr, l2 = LC.errors(y, ref)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (mr, l2)


def test_memory_cap_nomem(L):
    """A plan whose receive rows exceed the context's memory cap fails with LLEP_ERR_NOMEM (the Q3
    'tight memory cap' configuration), and the context stays usable under a larger cap."""
    sh = W.LayerShape(8, 2, 256, 512, 1024, 1)
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, 95, 1, 5, "cuda")
    ctx = L.Context(8, 2, 256, 512, 1, 0, 0, 1024)
    ctx.enable_backward()
    ctx.set_memory_cap(ctx.device_bytes() + 1024)   # nothing can grow
    dout = torch.zeros_like(x)
    with pytest.raises(L.LLEPError) as ei:
        plan, _ = ctx.prepare(ids)
        ctx.reserve(1 << 20, 4, 4)
    assert ei.value.code == 4
    ctx.set_memory_cap(0)
    out = ctx(x, ids, gates, w13, w2)
    torch.cuda.synchronize()
    ref = LC.oracle_rank_output(sh, 0, ids_np, g_np, 5)
    mr, l2 = LC.errors(out.float().cpu().numpy().astype(np.float64), ref)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2
    ctx.close()


def test_inconsistent_plan_rejected(L):
    """A plan whose chunk totals differ from the exchanged loads -> LLEP_ERR_PLAN."""
    sh = W.LayerShape(8, 2, 256, 512, 1024, 1)
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, 95, 1, 5, "cuda")
    ctx = L.Context(8, 2, 256, 512, 1, 0, 0, 1024)
    good, _ = ctx.prepare(ids)          # kept alive: plans are identified by address
    other = L.plan_host([100] * 8, 1, 1.0, 0, 1.0)
    bad = torch.frombuffer(bytearray(other.raw), dtype=torch.uint8).cuda()
    with pytest.raises(L.LLEPError) as ei:
        ctx.forward(x, ids, gates, w13, w2, bad)
    assert ei.value.code == 2
    ctx.forward(x, ids, gates, w13, w2, good)   # the prepared plan still works
    ctx.close()


def test_layer_trace_replay(L, tmp_path):
    """Row f4 (trace replay): one context replays three trace records (SPEC format) with different
    batch sizes and skews; each step's output vs O3 on that record's routing."""
    N, K, D, H = 8, 2, 256, 512
    f = tmp_path / "trace.csv"
    f.write_text("a,100,100,100,100,100,100,100,100\n"       # balanced, 400 tokens
                 "b,1500,10,10,10,10,10,0,0\n"             # one hot expert, 775 tokens
                 "c,0,0,0,0,0,0,0,6\n")                    # everything on the last expert, 3 tokens
    recs = W.load_trace(str(f), N, world=1)
    ctx = L.Context(N, K, D, H, 1, 0, 0, 1024)
    seed = 21
    w13, w2 = W.expert_weights_torch(range(N), D, H, "cuda", seed)
    x_all = W.tokens_torch(1024, D, 0, "cuda", seed)
    for rec in recs:
        ids_np = W.routing_from_counts(rec[0], K, 0, seed)
        B = ids_np.shape[0]
        g_np = W.gate_weights(B, K, 0, seed)
        out = ctx(x_all[:B].contiguous(), torch.from_numpy(ids_np).cuda(), torch.from_numpy(g_np).cuda(), w13, w2)
        torch.cuda.synchronize()
        ref = LC.oracle_rank_output(W.LayerShape(N, K, D, H, B, 1), 0, ids_np, g_np, seed)
        mr, l2 = LC.errors(_to_np(out), ref)
        assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (rec, mr, l2)
    ctx.close()


def test_multiprocess_trace_replay_p2(L, tmp_path):
    """Row f4 at P=2 (processes sharing cuda:0): replay the six records of a SPEC-format trace whose
    skew changes per record (tools/traces/tiny_mix_p2.csv, per-device counts) on one context per
    rank; every record's LLEP output vs O3 on that record's routing, and LLEP == EP bitwise."""
    trace = os.path.join(os.path.dirname(HERE), "tools", "traces", "tiny_mix_p2.csv")
    P = 2
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29561", LLEP_TEST_TRACE=trace)
    cmd = [sys.executable, os.path.join(HERE, "mp_layer_worker.py"), str(P), "tiny", "95", "1", str(tmp_path)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    sh0 = W.CONFIGS["tiny"]
    recs = W.load_trace(trace, sh0.n_experts, P)
    w = LC.OracleWeights(sh0.d_model, sh0.d_ff, 21)
    for p in range(P):
        res = np.load(os.path.join(tmp_path, f"rank{p}.npz"))
        assert int(res["n_records"]) == len(recs) == 6
        for i, C in enumerate(recs):
            ids = W.routing_from_counts(C[p], sh0.top_k, p, 21 + i)
            B = ids.shape[0]
            sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, B, P)
            ref = LC.oracle_rank_output(sh, p, ids, W.gate_weights(B, sh0.top_k, p, 21 + i), 21, weights=w)
            mr, l2 = LC.errors(res[f"r{i}_llep"].astype(np.float64), ref)
            assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (p, i, mr, l2)
            assert bool(res[f"r{i}_same"])


def test_peak_memory_bounded_by_plan(tmp_path):
    """G120 at P=8 (8 processes on one GPU, each holding exactly one GPU's footprint), 95 %/1: every
    rank's measured peak (torch allocations + the library context) stays within the §8(a) memory
    model at the plan's own g_a[d] and |S_d| plus a fixed 0.6 GB slack (scratch), and every rank's
    rows equal the capacity cap = B·K (the planner's constraint, α = 1)."""
    import json
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, os.path.join(os.path.dirname(HERE), "tools", "mem_sweep.py"), "--config", "g120",
           "--world", "8", "--scenarios", "95:1", "--modes", "llep", "--port", "29730"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    ll = line["llep"]
    assert ll["transfers"] == 7 and not ll["fallback"]
    assert ll["max_rows"] == W.CONFIGS["g120"].tokens_per_rank * W.CONFIGS["g120"].top_k
    assert ll["peak_gb_per_gpu"] <= ll["model_gb_critical"] + 0.6, ll
    assert ll["model_gb_critical"] < line["ep"]["model_gb_critical"] / 3


def test_forward_rejects_ids_other_than_prepared(L):
    """§8(b) boundary: llep_moe_forward runs the plan, load matrix and local ranks of the LAST
    llep_prepare.  A different topk_ids buffer with the same B -> LLEP_ERR_PLAN at once; the prepared
    buffer modified in place -> the changed slots are dropped (every other token's output is still
    exact) and llep_context_check reports LLEP_ERR_PLAN; the next prepare/forward is clean."""
    sh = W.LayerShape(8, 2, 256, 512, 1024, 1)
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, 95, 1, 5, "cuda")
    ctx = L.Context(8, 2, 256, 512, 1, 0, 0, 1024)
    plan, _ = ctx.prepare(ids)
    other = ids.clone()
    other[:, 0] = (other[:, 0] + 1) % 8
    with pytest.raises(L.LLEPError) as ei:
        ctx.forward(x, other, gates, w13, w2, plan)
    assert ei.value.code == 2
    ctx.check()                                   # nothing ran: no sticky error
    # in-place change of the prepared buffer after prepare: tokens 0..9 slot 1 -> another expert
    ids_new = ids_np.copy()
    ids_new[:10, 1] = (ids_new[:10, 1] + 3) % 8
    ids.copy_(torch.from_numpy(ids_new).cuda())
    out = ctx.forward(x, ids, gates, w13, w2, plan)
    with pytest.raises(L.LLEPError) as ei:
        ctx.check()
    assert ei.value.code == 2
    ctx.check()                                   # reported once, then cleared
    y = _to_np(out)
    g_drop = g_np.copy()
    g_drop[:10, 1] = 0.0                          # the changed slots contribute nothing
    ref = LC.oracle_rank_output(sh, 0, ids_np, g_drop, 5)
    mr, l2 = LC.errors(y, ref)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (mr, l2)
    # a fresh prepare on the new ids gives the exact output of the new routing
    out2 = ctx(x, ids, gates, w13, w2)
    ctx.check()
    ref2 = LC.oracle_rank_output(sh, 0, ids_new, g_np, 5)
    mr, l2 = LC.errors(_to_np(out2), ref2)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (mr, l2)
    ctx.close()


def test_asymmetric_arenas_rejected(tmp_path):
    """ADVICE r1 (symmetric arena): two ranks whose contexts were created with different max_tokens
    (raw C ABI, bypassing the binding's max-over-ranks) -> llep_context_open_peers fails with
    LLEP_ERR_INVALID on both ranks instead of mapping arenas whose regions sit at different offsets."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29571")
    cmd = [sys.executable, os.path.join(HERE, "mp_asym_worker.py"), str(tmp_path)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    codes = [int(np.load(os.path.join(tmp_path, f"asym{p}.npy"))) for p in range(2)]
    assert codes == [1, 1], codes


def test_nccl_all_to_all_crosscheck(tmp_path):
    """on >= 2 GPUs, the rows the NVLink peer-store dispatch wrote into every device's receive
    arena equal, bit for bit, the rows torch.distributed.all_to_all_single (NCCL) delivers for the same
    plan.  Skips on a one-GPU box (the data plane then runs as processes sharing one GPU, covered above)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs for NCCL")
    P = min(torch.cuda.device_count(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", "29587",
           os.path.join(HERE, "mp_nccl_xcheck_worker.py"), str(tmp_path), "g120", "95", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for p in range(P):
        res = np.load(os.path.join(tmp_path, f"xcheck{p}.npz"))
        assert int(res["rows"]) > 0 and bool(res["same"]), (p, res["sent"], res["received"])


def test_dispatch_overlap_matches_barrier(L, tmp_path):
    """Row f2: the dispatch overlapped with GEMM1 through per-source arrival flags gives bit-identical
    outputs to the old dispatch -> barrier -> GEMM1 order (LLEP_DISPATCH_BARRIER=1), at P=4 with spills."""
    outs = {}
    for mode in ("overlap", "barrier"):
        d = tmp_path / mode
        d.mkdir()
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29575 + len(mode)))
        if mode == "barrier":
            env["LLEP_DISPATCH_BARRIER"] = "1"
        cmd = [sys.executable, os.path.join(HERE, "mp_layer_worker.py"), "4", "tiny", "80", "1", str(d)]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        outs[mode] = [np.load(os.path.join(d, f"rank{p}.npz"))["llep"] for p in range(4)]
    for a, b in zip(outs["overlap"], outs["barrier"]):
        assert np.array_equal(a, b)


def _few_expert_rows(ids_np, n_experts_max, head=40, tail=24):
    """Tokens whose K experts all lie in 0..n_experts_max-1 (the hot expert and a few cold ones), the
    first `head` and last `tail` of them: few experts' weights for the float64 oracle."""
    ok = np.nonzero((ids_np < n_experts_max).all(1))[0]
    return np.unique(np.concatenate([ok[:head], ok[-tail:]]))


@pytest.mark.parametrize("cfg", ["dsv3", "kimi", "fhead"])
def test_f3_shapes_p1_sampled_parity(L, cfg):
    """Row f3: the paper's other layer shapes at P=1, 95 %/1 -- DeepSeek-V3 (N=256, K=8, D=7168, H=2048,
    16K), Kimi-K2 (N=384, same dims) (F-models) and the F-head layer (N=128, K=4, D=H=2048,
    32K): sampled outputs vs O3 and the index work (a1, a3, a5) bit-exact vs O2."""
    from oracle import planner as O1
    from oracle import schedule as O2
    import mp_layer_worker as MW
    sh0 = W.CONFIGS[cfg]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, 1)
    seed = 43
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, 95, 1, seed, "cuda")
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, 1, 0, 0, sh.tokens_per_rank)
    out = ctx(x, ids, gates, w13, w2)
    ctx.check()
    res = [MW.dump_index_work(L, ctx, sh, 1, "llep")]
    LC.check_index_work(res, "llep", O1.plan(O2.local_counts(ids_np, sh.n_experts).tolist(), 1), [ids_np],
                        sh.n_experts)
    rows = _few_expert_rows(ids_np, 12)
    y = _to_np(out[torch.from_numpy(rows).cuda()])
    ctx.close()
    del out, w13, w2
    ref = LC.oracle_rank_output(sh, 0, ids_np, g_np, seed, rows=rows)
    mr, l2 = LC.errors(y, ref)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (cfg, mr, l2)


def test_f3_dsv3_p4_processes(L, tmp_path):
    """Row f3 at EP 4: the DeepSeek-V3-shaped layer (N=256, K=8, D=7168, H=2048, 16K tokens/rank), 95 %/1,
    four processes sharing cuda:0.  Plan == O1 on every rank, index work bit-exact vs O2 for LLEP and
    EP, sampled outputs vs O3 (tokens whose experts all lie in 0..11), LLEP == EP bitwise."""
    from oracle import planner as O1
    from oracle import schedule as O2
    P, cfg = 4, "dsv3"
    sh0 = W.CONFIGS[cfg]
    sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, P)
    ids_all = [W.routing_ids(sh, p, 95, 1, 21) for p in range(P)]
    C = O2.load_matrix(ids_all, sh.n_experts)
    ref_plan = O1.plan(C.sum(0).tolist(), P)
    rows = {p: _few_expert_rows(ids_all[p], 12, 16, 8) for p in range(P)}
    rows_file = os.path.join(tmp_path, "rows.npz")
    np.savez(rows_file, **{f"r{p}": rows[p] for p in range(P)})
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29591", LLEP_TEST_ROWS=rows_file)
    cmd = [sys.executable, os.path.join(HERE, "mp_layer_worker.py"), str(P), cfg, "95", "1", str(tmp_path)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"rank{p}.npz")) for p in range(P)]
    dp = L.parse_plan(bytes(res[0]["plan"].tobytes()))
    assert [list(A) for A in dp.chunks] == [list(A) for A in ref_plan.chunks] and len(ref_plan.transfers) > 0
    LC.check_index_work(res, "llep", ref_plan, ids_all, sh.n_experts)
    LC.check_index_work(res, "ep", O1.ep_plan(C.sum(0).tolist(), P, 1.0, fallback=False), ids_all, sh.n_experts)
    w = LC.OracleWeights(sh.d_model, sh.d_ff, 21)
    for p in range(P):
        ref = LC.oracle_rank_output(sh, p, ids_all[p], W.gate_weights(sh.tokens_per_rank, sh.top_k, p, 21), 21,
                                    rows=rows[p], weights=w)
        mr, l2 = LC.errors(res[p]["llep"].astype(np.float64), ref)
        assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (p, mr, l2)
        assert bool(res[p]["same"])


@pytest.mark.parametrize("cfg,pct,nhot", [("tiny", 95, 1), ("tiny", None, 0), ("tiny", 50, 4), ("g20", 95, 1)])
def test_local_gather_bitwise_equals_copy(L, cfg, pct, nhot):
    """a6 local rows (opt-in LLEP_GATHER=1): GEMM1 gathering this rank's own rows from x (TMA gather4, no
    dispatch copy) gives bit-identical outputs and saved [g | u] to the default copy into the receive
    buffer: same A tiles in shared memory, same MMAs.  Covers full, half and swapped tiles."""
    base = W.CONFIGS[cfg]
    B = min(base.tokens_per_rank, 4096)
    sh = W.LayerShape(base.n_experts, base.top_k, base.d_model, base.d_ff, B, 1)
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, pct, nhot, 13, "cuda")
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, 1, 0, 0, B)
    res = {}
    for mode in ("gather", "copy"):
        if mode == "gather":
            os.environ["LLEP_GATHER"] = "1"
        try:
            plan, req = ctx.prepare(ids)
            out = ctx.forward(x, ids, gates, w13, w2, plan)
            gu = torch.zeros((int(req.rows_needed), 2 * sh.d_ff), dtype=torch.bfloat16, device="cuda")
            out2, gu = ctx.forward_train(x, ids, gates, w13, w2, plan, gu=gu)
            torch.cuda.synchronize()
            res[mode] = (out.cpu(), out2.cpu(), gu.cpu())
        finally:
            os.environ.pop("LLEP_GATHER", None)
    for a, b in zip(res["gather"], res["copy"]):
        assert torch.equal(a, b)
    ref = LC.oracle_rank_output(sh, 0, ids_np, g_np, 13, rows=np.arange(min(B, 256)))
    mr, l2 = LC.errors(_to_np(res["gather"][0][: min(B, 256)]), ref)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (mr, l2)
    ctx.close()


def test_token_orders_same_outputs_different_rows(L, tmp_path):
    """a3/a5 token order (llep_context_set_token_order): the rank-major order (R11) and the default
    chunk-aligned one (R11') give bit-identical outputs (each row is computed alone, the K-sum is in slot
    order) with each order's index work bit-exact vs O2 at P=4 with spills; the aligned order keeps more
    of the spilled rows on their own rank."""
    from oracle import planner as O1
    from oracle import schedule as O2
    outs, dst = {}, {}
    for order in ("rank_major", "chunk_aligned"):
        d = tmp_path / order
        d.mkdir()
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29585 + len(order)), LLEP_TEST_ORDER=order)
        cmd = [sys.executable, os.path.join(HERE, "mp_layer_worker.py"), "4", "tiny", "95", "1", str(d)]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        res = [np.load(os.path.join(d, f"rank{p}.npz")) for p in range(4)]
        sh0 = W.CONFIGS["tiny"]
        sh = W.LayerShape(sh0.n_experts, sh0.top_k, sh0.d_model, sh0.d_ff, sh0.tokens_per_rank, 4)
        ids_all = [W.routing_ids(sh, p, 95, 1, 21) for p in range(4)]
        C = O2.load_matrix(ids_all, sh.n_experts)
        plan = O1.plan(C.sum(0).tolist(), 4)
        LC.check_index_work(res, "llep", plan, ids_all, sh.n_experts, aligned=(order == "chunk_aligned"))
        outs[order] = [r_["llep"] for r_ in res]
        dst[order] = sum(int((r_["llep_dst"][:, 0] == p).sum()) for p, r_ in enumerate(res))
    for a, b in zip(outs["rank_major"], outs["chunk_aligned"]):
        assert np.array_equal(a, b)
    assert dst["chunk_aligned"] > dst["rank_major"], dst


@pytest.mark.parametrize("cfg", ["g20", "q3"])
def test_multicast_clusters_bitwise_equal(L, cfg):
    """Opt-in two-pair clusters with the activation tile multicast (LLEP_GEMM_MC=2) give bit-identical
    layer outputs and saved [g | u] to the default single-pair kernels: same tiles, same MMAs, same K order."""
    base = W.CONFIGS[cfg]
    B = min(base.tokens_per_rank, 4096)
    sh = W.LayerShape(base.n_experts, base.top_k, base.d_model, base.d_ff, B, 1)
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, 95, 1, 17, "cuda")
    ctx = L.Context(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, 1, 0, 0, B)
    res = {}
    for mc in ("1", "2"):
        os.environ["LLEP_GEMM_MC"] = mc
        try:
            plan, req = ctx.prepare(ids)
            out = ctx.forward(x, ids, gates, w13, w2, plan)
            gu = torch.zeros((int(req.rows_needed), 2 * sh.d_ff), dtype=torch.bfloat16, device="cuda")
            out2, gu = ctx.forward_train(x, ids, gates, w13, w2, plan, gu=gu)
            torch.cuda.synchronize()
            res[mc] = (out.cpu(), out2.cpu(), gu.cpu())
        finally:
            os.environ.pop("LLEP_GEMM_MC", None)
    for a, b in zip(res["1"], res["2"]):
        assert torch.equal(a, b)
    ctx.close()
