"""Pins for O2 (schedule), O3 (layer) and O4 (simulated EP / LLEP) -- CPU only."""
import json
import math
import os
import random

import numpy as np
import pytest

from oracle import layer as O3
from oracle import planner as O1
from oracle import schedule as O2
from oracle import simulate as O4
from synth import workload as W


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ O2
def test_reindex_worked_examples(golden_dir):
    g = _load(golden_dir, "schedule_examples.json")
    ex = g["reindex"][0]
    ids = np.array(ex["ids"])
    perm, sorted_ids = O2.stable_reindex(ids)
    assert perm.tolist() == ex["sorted_tokens"]
    cnt = O2.local_counts(ids, ex["n_experts"])
    assert {str(e): int(c) for e, c in enumerate(cnt) if c} == ex["counts"]
    ex = g["reindex"][1]
    ids = np.array(ex["ids"])
    perm, sorted_ids = O2.stable_reindex(ids)
    assert perm[sorted_ids == 0].tolist() == ex["expert0_flat_slots"]
    r = O2.local_rank_in_expert(ids)
    assert r.tolist() == [0, 0, 1, 1, 2, 2]


def test_materialize_example(golden_dir):
    ex = _load(golden_dir, "schedule_examples.json")["materialize"][0]
    C = np.array(ex["C"])
    plan = O1.Plan(2, 2, [[tuple(c) for c in A] for A in ex["chunks"]], [5, 5], 5, 10, False)
    sch = O2.send_schedule(plan, C)
    for key, sl in ex["slices"].items():
        p, e = map(int, key.split(","))
        assert [list(s) for s in sch[(p, e)]] == sl


def test_global_index_rank_major_worked_example(golden_dir):
    """R11 / S:253 (rank-major global order): expert e0 has counts [6, 4] on ranks 0 and 1, so rank 0's
    six slots of e0 take global indices 0..5 and rank 1's four take 6..9 (a reversed rank order,
    Σ_{q>p}, would give rank 0 indices 4..9).  Under S:253's plan e0 -> [(0,0,5),(1,5,10)], rank 0's
    local [0,5) goes to device 0 rows 0..4, its local [5,6) to device 1 row 0, and rank 1's local
    [0,4) to device 1 rows 1..4 (chunks of e0 on device 1 concatenated in plan order)."""
    ex = _load(golden_dir, "schedule_examples.json")["materialize"][0]
    C = np.array(ex["C"])
    # K = 1: rank 0 holds six tokens routed to e0, rank 1 four (C's e1 column is empty)
    ids0 = np.array([[0], [0], [0], [0], [0], [0]])
    ids1 = np.array([[0], [0], [0], [0]])
    assert O2.global_index(ids0, C, 0).tolist() == [0, 1, 2, 3, 4, 5]
    assert O2.global_index(ids1, C, 1).tolist() == [6, 7, 8, 9]
    plan = O1.Plan(2, 2, [[tuple(c) for c in A] for A in ex["chunks"]], [5, 5], 5, 10, False)
    d0, r0 = O2.slot_destinations(plan, C, ids0, 0)
    d1, r1 = O2.slot_destinations(plan, C, ids1, 1)
    assert d0.tolist() == [0, 0, 0, 0, 0, 1] and r0.tolist() == [0, 1, 2, 3, 4, 0]
    assert d1.tolist() == [1, 1, 1, 1] and r1.tolist() == [1, 2, 3, 4]
    # with K = 2 and other experts interleaved the index counts only e's own earlier slots
    C2 = np.array([[2, 3], [1, 2]])
    ids_r1 = np.array([[1, 0], [1, 1]])     # flat slots: e1, e0, e1, e1
    assert O2.global_index(ids_r1, C2, 1).tolist() == [3, 2, 4, 5]


def test_relative_errors_hand_values():
    """R21: max_rel = max|y-r| / max|r| and rel_L2 = ||y-r||_2 / ||r||_2 over the WHOLE output.
    y=[1,2], r=[1,1]: diff [0,1] -> max_rel 1, rel_L2 1/sqrt(2).  y=[2,0], r=[4,2]: max_rel 2/4 (a
    y-normaliser would give 1), rel_L2 sqrt(8/20).  2-D: the max is over all elements, not per row
    (a per-row normaliser would give 1 for the first row)."""
    mr, l2 = O3.relative_errors(np.array([1.0, 2.0]), np.array([1.0, 1.0]))
    assert mr == 1.0 and l2 == pytest.approx(1 / math.sqrt(2), rel=1e-15)
    mr, l2 = O3.relative_errors(np.array([2.0, 0.0]), np.array([4.0, 2.0]))
    assert mr == 0.5 and l2 == pytest.approx(math.sqrt(0.4), rel=1e-15)
    mr, l2 = O3.relative_errors(np.array([[1.0, 0.0], [10.0, 10.0]]), np.array([[1.0, 1.0], [10.0, 10.0]]))
    assert mr == 0.1 and l2 == pytest.approx(1 / math.sqrt(202), rel=1e-15)
    assert O3.relative_errors(np.array([3.0, -4.0]), np.array([3.0, -4.0])) == (0.0, 0.0)


def test_out_of_range_ids():
    with pytest.raises(ValueError):
        O2.local_counts(np.array([[0, 5]]), 4)


def _check_destinations(plan, C, ids_per_rank):
    """Every (token, slot) pair lands exactly once; per (e, d) positions are 0..rows-1."""
    seen = {}
    for p, ids in enumerate(ids_per_rank):
        dev, pos = O2.slot_destinations(plan, C, ids, p)
        flat = ids.reshape(-1)
        for j in range(flat.size):
            key = (int(flat[j]), int(dev[j]))
            seen.setdefault(key, []).append(int(pos[j]))
    for e in range(plan.n_experts):
        for d in range(plan.world):
            n = O2.rows_on_device(plan, e, d)
            got = sorted(seen.get((e, d), []))
            assert got == list(range(n)), (e, d)


def test_destinations_fuzz():
    rng = np.random.default_rng(7)
    for trial in range(60):
        P = int(rng.choice([1, 2, 3, 4]))
        M = int(rng.integers(1, 4))
        N = P * M
        K = int(rng.integers(1, 4))
        B = int(rng.integers(0, 40))
        hot = int(rng.integers(0, N))
        ids = []
        for p in range(P):
            x = rng.integers(0, N, size=(B, K))
            x[rng.random((B, K)) < 0.6] = hot
            ids.append(x.astype(np.int32))
        C = O2.load_matrix(ids, N)
        plan = O1.plan(C.sum(0).tolist(), P, 1.0, int(rng.choice([0, 1, 3, 50])), 1.0)
        _check_destinations(plan, C, ids)
        # schedule consistency: destination totals per (e, d) == chunk sizes
        sch = O2.send_schedule(plan, C)
        for e in range(N):
            for d in range(P):
                tot = sum(b - a for p in range(P) for (dd, a, b) in sch[(p, e)] if dd == d)
                assert tot == O2.rows_on_device(plan, e, d)


# ------------------------------------------------------------------ O3
def test_linear_hand_value():
    """D=2, N=2, K=1, u=[1,0], gate 0.8808, W_0 = [[1],[1]] (H=1) -> h = 0.8808."""
    x = np.array([[1.0, 0.0]])
    ids = np.array([[0]])
    g = np.array([[0.8808]])
    Ws = {0: np.array([[1.0], [1.0]]), 1: np.array([[5.0], [7.0]])}
    h = O3.moe_forward_linear(x, ids, g, lambda e: Ws[e])
    assert h.shape == (1, 1) and h[0, 0] == pytest.approx(0.8808, abs=1e-15)


def test_swiglu_hand_values():
    """1-D SwiGLU: u=2, w_gate=ln3/2 -> z=ln 3, silu(ln 3) = ln3 · 3/4 (sigmoid(ln 3) = 3/4);
    w_up=5 -> 10; w_down=0.5 -> FFN = 0.5 · 0.75 ln3 · 10 = 3.75 ln 3.  Swapping gate/up, a sign
    error in the sigmoid or dropping W_down all change the value."""
    w = (np.array([[math.log(3) / 2]]), np.array([[5.0]]), np.array([[0.5]]))
    y = O3.swiglu_ffn(np.array([[2.0]]), w)
    assert y[0, 0] == pytest.approx(3.75 * math.log(3), rel=1e-14)
    # 2-D case: orientation of W_gate [H, D], W_up [H, D], W_down [D, H] (D=2, H=1)
    wg = np.array([[math.log(3), 0.0]])       # z = ln3 · u0
    wu = np.array([[0.0, 2.0]])               # up = 2 · u1
    wd = np.array([[1.0], [-3.0]])            # out = [a, -3a]
    y = O3.swiglu_ffn(np.array([[1.0, 4.0]]), (wg, wu, wd))
    a = 0.75 * math.log(3) * 8.0
    assert y[0].tolist() == pytest.approx([a, -3 * a], rel=1e-14)


def _rand_weights(rng, D, H):
    return (rng.standard_normal((H, D)) / np.sqrt(D), rng.standard_normal((H, D)) / np.sqrt(D),
            rng.standard_normal((D, H)) / np.sqrt(H))


def test_layer_special_cases():
    rng = np.random.default_rng(3)
    D, H, N = 8, 6, 4
    Ws = {e: _rand_weights(rng, D, H) for e in range(N)}
    # zero token -> 0
    out = O3.moe_forward(np.zeros((2, D)), np.array([[0, 1], [2, 3]]), np.ones((2, 2)), Ws.get)
    assert np.all(out == 0)
    # gate 0 -> no contribution; all K slots on one expert with gates summing to 1 -> one FFN
    x = rng.standard_normal((3, D))
    out = O3.moe_forward(x, np.array([[1, 1, 1]] * 3), np.array([[0.25, 0.5, 0.25]] * 3), Ws.get)
    ref = O3.swiglu_ffn(x, Ws[1])
    np.testing.assert_allclose(out, ref, rtol=1e-14, atol=1e-15)
    out2 = O3.moe_forward(x, np.array([[1, 2, 1]] * 3), np.array([[0.5, 0.0, 0.5]] * 3), Ws.get)
    np.testing.assert_allclose(out2, ref, rtol=1e-14, atol=1e-15)


def test_layer_linearity_in_gates():
    """Eq. 1 is linear in the gates: out(g1 + g2) = out(g1) + out(g2)."""
    rng = np.random.default_rng(4)
    D, H, N, T, K = 16, 8, 5, 12, 3
    Ws = {e: _rand_weights(rng, D, H) for e in range(N)}
    x = rng.standard_normal((T, D))
    ids = rng.integers(0, N, (T, K))
    g1, g2 = rng.random((T, K)), rng.random((T, K))
    a = O3.moe_forward(x, ids, g1 + g2, Ws.get)
    b = O3.moe_forward(x, ids, g1, Ws.get) + O3.moe_forward(x, ids, g2, Ws.get)
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ O4
def _sim_case(rng, P, M, K, B, D, H, hot_share, m, lam):
    N = P * M
    Ws = {e: _rand_weights(rng, D, H) for e in range(N)}
    xs, ids, gs = [], [], []
    for p in range(P):
        xs.append(rng.standard_normal((B, D)))
        i = rng.integers(0, N, (B, K))
        i[rng.random((B, K)) < hot_share] = 0
        ids.append(i)
        gs.append(rng.random((B, K)))
    return N, Ws, xs, ids, gs


@pytest.mark.parametrize("seed", range(12))
def test_ep_llep_dense_equal(seed):
    """Exactness: LLEP == EP == dense Eq. 1 within 1e-12 relative, incl. duplicate ids,
    zero-load experts, force-assign plans and the λ fallback."""
    rng = np.random.default_rng(100 + seed)
    P = [1, 2, 3, 4][seed % 4]
    M = 1 + seed % 3
    K = 1 + seed % 3
    B = 5 + 3 * seed
    N, Ws, xs, ids, gs = _sim_case(rng, P, M, K, B, 6, 5, [0.0, 0.5, 0.9][seed % 3], [0, 2, 7][seed % 3],
                                   [1.0, 1.3][seed % 2])
    dense = [O3.moe_forward(xs[p], ids[p], gs[p], Ws.get) for p in range(P)]
    ep, _, _ = O4.dispatch_combine(xs, ids, gs, Ws.get, N, P, mode="ep")
    ll, plan, _ = O4.dispatch_combine(xs, ids, gs, Ws.get, N, P, mode="llep",
                                      min_chunk=[0, 2, 7][seed % 3], lam=[1.0, 1.3][seed % 2])
    scale = max(np.abs(d).max() for d in dense)
    for p in range(P):
        assert np.abs(ep[p] - dense[p]).max() <= 1e-12 * scale
        assert np.abs(ll[p] - dense[p]).max() <= 1e-12 * scale


def test_llep_spills_and_forces_are_exercised():
    rng = np.random.default_rng(9)
    seen_force = seen_transfer = False
    for t in range(30):
        N, Ws, xs, ids, gs = _sim_case(rng, 3, 2, 2, 15, 4, 3, 0.6, 20, 1.0)
        dense = [O3.moe_forward(xs[p], ids[p], gs[p], Ws.get) for p in range(3)]
        ll, plan, st = O4.dispatch_combine(xs, ids, gs, Ws.get, N, 3, mode="llep", min_chunk=20, lam=1.0)
        seen_force |= plan.force_count > 0
        seen_transfer |= len(plan.transfers) > 0
        for p in range(3):
            np.testing.assert_allclose(ll[p], dense[p], rtol=1e-12, atol=1e-12)
    assert seen_force and seen_transfer


def test_workload_shapes_and_slot_fractions():
    """The synthetic scenario: hot ids 0..y-1 get x/y of all slots each."""
    sh = W.CONFIGS["g120"]
    for pct, y in [(95, 1), (50, 4), (30, 16)]:
        c = W.slot_counts(sh.n_experts, sh.tokens_per_rank * sh.top_k, pct, y)
        assert c.sum() == sh.tokens_per_rank * sh.top_k
        hot = c[:y].sum() / c.sum()
        assert abs(hot - pct / 100) < 1e-4
        assert c[:y].max() - c[:y].min() <= 1 and c[y:].max() - c[y:].min() <= 1
    ids = W.routing_ids(W.CONFIGS["tiny"], 0, 95, 1)
    assert ids.shape == (1024, 2) and ids.dtype == np.int32
    assert np.bincount(ids.ravel(), minlength=8).tolist() == W.slot_counts(8, 2048, 95, 1).tolist()
    g = W.gate_weights(16, 4, 0)
    assert np.all(g > 0) and np.allclose(g.sum(1), 1.0, atol=1e-6)


def test_generator_numpy_torch_identical():
    """The counter-based generator gives identical bf16 bits on numpy and torch (CPU here)."""
    import torch
    bits = W.tokens_bits(7, 33, 3)
    t = W.tokens_torch(7, 33, 3, "cpu")
    assert np.array_equal(t.view(torch.int16).numpy().view(np.uint16), bits)
    rows = W.token_rows_bits(np.array([5, 0, 2]), 33, 3)
    assert np.array_equal(rows, bits[[5, 0, 2]])
    wg, wu, wd = W.expert_weights_bits(5, 24, 16)
    w13, w2 = W.expert_weights_torch([5], 24, 16, "cpu")
    assert np.array_equal(w13[0, :16].view(torch.int16).numpy().view(np.uint16), wg)
    assert np.array_equal(w13[0, 16:].view(torch.int16).numpy().view(np.uint16), wu)
    assert np.array_equal(w2[0].view(torch.int16).numpy().view(np.uint16), wd)
    # bf16 RNE rounding matches torch's conversion on awkward values
    f = np.array([1.0, 1.00390625, 1.01171875, -3.0e-39, 65504.0, 1e30], dtype=np.float32)
    assert np.array_equal(W.bf16_bits_from_f32(f),
                          torch.from_numpy(f).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16))


def test_distinct_routing_generator():
    """SPEC generate_routing: K distinct ids per token by weighted sampling without replacement.
    With K=1 it is plain categorical sampling, so the hot expert's share approaches x (95 %); with K=4 a
    token can hold the hot expert once, so its share is capped at 1/K; deterministic per seed."""
    sh1 = W.LayerShape(128, 1, 64, 64, 20000, 1)
    ids = W.routing_ids(sh1, 0, 95, 1, distinct=True)
    assert abs((ids == 0).mean() - 0.95) < 0.01
    sh = W.LayerShape(128, 4, 64, 64, 4096, 1)
    ids = W.routing_ids(sh, 0, 95, 1, distinct=True)
    assert ids.shape == (4096, 4) and ids.dtype == np.int32
    assert all(len(set(r.tolist())) == 4 for r in ids)
    assert (ids == 0).any(axis=1).mean() > 0.99 and (ids == 0).mean() <= 0.25
    assert np.array_equal(ids, W.routing_ids(sh, 0, 95, 1, distinct=True))
    bal = W.routing_ids(W.LayerShape(8, 2, 64, 64, 40000, 1), 0, None, 0, distinct=True)
    c = np.bincount(bal.ravel(), minlength=8)
    assert np.all(np.abs(c - 10000) < 5 * np.sqrt(10000))


def _loop_local_rank(flat):
    seen, r = {}, []
    for e in flat.tolist():
        r.append(seen.get(e, 0))
        seen[e] = seen.get(e, 0) + 1
    return r


def _loop_destinations(plan, C, flat, rank):
    """Slot-by-slot transcription of S:247-255 (independent of O2's vectorised form)."""
    before = [int(C[:rank, e].sum()) for e in range(C.shape[1])]
    seen, dev, pos = {}, [], []
    for e in flat.tolist():
        g = before[e] + seen.get(e, 0)
        seen[e] = seen.get(e, 0) + 1
        off = {}
        for (d0, s, t) in plan.chunks[e]:
            if s <= g < t:
                dev.append(d0)
                pos.append(off.get(d0, 0) + g - s)
                break
            off[d0] = off.get(d0, 0) + t - s
    return dev, pos


def test_schedule_vectorised_equals_slot_loop():
    """O2's local ranks and destinations equal a plain per-slot loop (counting seen slots, walking the
    chunks) on random plans with spills, forces, zero-load experts and duplicate ids."""
    rng = np.random.default_rng(17)
    for trial in range(80):
        P = int(rng.choice([1, 2, 3, 4, 8]))
        N = P * int(rng.integers(1, 5))
        K = int(rng.integers(1, 5))
        ids = []
        for p in range(P):
            x = rng.integers(0, N, size=(int(rng.integers(0, 60)), K))
            x[rng.random(x.shape) < 0.5] = int(rng.integers(0, N))
            ids.append(x.astype(np.int32))
        C = O2.load_matrix(ids, N)
        plan = O1.plan(C.sum(0).tolist(), P, float(rng.choice([1.0, 1.5])), int(rng.choice([0, 2, 9])), 1.0)
        for p in range(P):
            flat = ids[p].reshape(-1)
            assert O2.local_rank_in_expert(flat).tolist() == _loop_local_rank(flat)
            dev, pos = O2.slot_destinations(plan, C, ids[p], p)
            d2, p2 = _loop_destinations(plan, C, flat, p)
            assert dev.tolist() == d2 and pos.tolist() == p2


def test_chunk_aligned_order_worked_example():
    """R11' by hand.  P=3, N=3 (M=1), K=1, loads l = [9, 2, 1] with e0's 9 slots split 3/3/3 over the
    ranks.  cap = floor(12/3) = 4; e0: native chunk (0, 0, 4), then LLAS picks the least-loaded device 2
    (load 1 < device 1's 2): (2, 4, 7), then device 1: (1, 7, 9).  Chunk-aligned source order of e0 =
    [0, 2, 1]: rank 0 takes global [0, 3), rank 2 [3, 6), rank 1 [6, 9) -- so rank 2's e0 slots land at
    4, 5 on device 2 (local) and rank 1's at 7, 8 on device 1 (local); rank-major would send all of
    rank 1's and two of rank 2's e0 slots across."""
    ids = [np.array([[0], [0], [0], [1]]), np.array([[0], [1], [0], [0]]), np.array([[0], [0], [2], [0]])]
    C = O2.load_matrix(ids, 3)
    assert C[:, 0].tolist() == [3, 3, 3] and C.sum(0).tolist() == [9, 2, 1]
    plan = O1.plan(C.sum(0).tolist(), 3, 1.0, 1, 1.3)
    assert plan.chunks[0] == [(0, 0, 4), (2, 4, 7), (1, 7, 9)]
    assert O2.source_order(plan, 0) == [0, 2, 1]
    assert O2.source_order(plan, 2) == [0, 1, 2]                 # one chunk: rank-major
    g = [O2.global_index(ids[p], C, p, plan) for p in range(3)]
    e0 = [g[p][ids[p].reshape(-1) == 0].tolist() for p in range(3)]
    assert e0 == [[0, 1, 2], [6, 7, 8], [3, 4, 5]]
    d = [O2.slot_destinations(plan, C, ids[p], p, aligned=True)[0] for p in range(3)]
    d_e0 = [d[p][ids[p].reshape(-1) == 0].tolist() for p in range(3)]
    assert d_e0 == [[0, 0, 0], [2, 1, 1], [0, 2, 2]]
    rm = [O2.slot_destinations(plan, C, ids[p], p)[0][ids[p].reshape(-1) == 0].tolist() for p in range(3)]
    assert rm == [[0, 0, 0], [0, 2, 2], [2, 1, 1]]
    local = lambda dd: sum(int(x == p) for p, row in enumerate(dd) for x in row)   # noqa: E731
    assert local(d_e0) == 7 and local(rm) == 4


def test_chunk_aligned_order_is_a_permutation_fuzz():
    """R11' covers every slot exactly once: per expert the aligned global indices of all ranks are a
    permutation of [0, l_e), each chunk receives exactly its rows, and experts with <= 1 chunk keep
    rank-major indices."""
    rng = np.random.default_rng(7)
    for it in range(300):
        P = int(rng.choice([2, 3, 4, 8]))
        M = int(rng.choice([1, 2, 4]))
        N, K = P * M, int(rng.integers(1, 4))
        B = int(rng.integers(0, 40))
        hot = rng.random(N) ** 4
        ids = [rng.choice(N, size=(B, K), p=hot / hot.sum()).astype(np.int32) for _ in range(P)]
        C = O2.load_matrix(ids, N)
        plan = O1.plan(C.sum(0).tolist(), P, float(rng.choice([1.0, 1.2])), int(rng.integers(0, 8)), 1.0)
        ga = [O2.global_index(ids[p], C, p, plan) for p in range(P)]
        gr = [O2.global_index(ids[p], C, p) for p in range(P)]
        for e in range(N):
            got = np.sort(np.concatenate([ga[p][ids[p].reshape(-1) == e] for p in range(P)]))
            assert got.tolist() == list(range(int(C[:, e].sum()))), (it, e)
            if len(plan.chunks[e]) <= 1:
                for p in range(P):
                    m = ids[p].reshape(-1) == e
                    assert np.array_equal(ga[p][m], gr[p][m])
        per_dev = np.zeros((N, P), dtype=np.int64)
        for p in range(P):
            dev, _pos = O2.slot_destinations(plan, C, ids[p], p, aligned=True)
            np.add.at(per_dev, (ids[p].reshape(-1), dev), 1)
        for e in range(N):
            for d in range(P):
                assert per_dev[e, d] == O2.rows_on_device(plan, e, d)


def test_chunk_aligned_order_keeps_g120_spills_local():
    """At the north-star layer shape (G120, P=8, 95 %/1, equal counts on every rank) the hot expert has a
    chunk on every device, in LLAS order (least loaded first, not rank order); under R11' each device's
    chunk is (almost) its own rows: > 99 % of the hot expert's slots stay on their rank, against ~1/8
    rank-major."""
    P = 8
    base = W.CONFIGS["g120"]
    sh = W.LayerShape(base.n_experts, base.top_k, base.d_model, base.d_ff, 4096, P)
    ids = [W.routing_ids(sh, p, 95, 1, 21) for p in range(P)]
    C = O2.load_matrix(ids, sh.n_experts)
    plan = O1.plan(C.sum(0).tolist(), P)
    order = [d for (d, _s, _t) in plan.chunks[0]]
    assert sorted(order) == list(range(P)) and order != list(range(P))
    frac = {}
    for aligned in (False, True):
        loc = tot = 0
        for p in range(P):
            dev, _ = O2.slot_destinations(plan, C, ids[p], p, aligned=aligned)
            m = ids[p].reshape(-1) == 0
            loc += int((dev[m] == p).sum())
            tot += int(m.sum())
        frac[aligned] = loc / tot
    assert frac[True] > 0.99 and frac[False] < 0.15, frac
