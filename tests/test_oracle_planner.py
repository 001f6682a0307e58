"""Pins for O1 (oracle/planner.py) against what the paper and arithmetic fix -- CPU only."""
import itertools
import json
import math
import os
import random

import numpy as np
import pytest

from oracle import planner as O1
from synth import workload as W


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ invariants
def check_invariants(l, P, alpha, m, plan, lam=None):
    """Plan invariants (north star): coverage, contiguity, conservation,
    native-first, capacity when no force, weight-plan soundness, chunk count bound."""
    N = len(l)
    M = N // P
    ga = [0] * P
    for e in range(N):
        A = plan.chunks[e]
        if l[e] == 0:
            assert A == []
            continue
        # coverage + contiguity: chunks nonempty, consecutive, [0, l_e)
        assert A[0][1] == 0 and A[-1][2] == l[e]
        for (d, s, t) in A:
            assert 0 <= d < P and s < t
            ga[d] += t - s
        for a, b in zip(A, A[1:]):
            assert a[2] == b[1]
        assert len(A) <= P + 1
    assert ga == plan.assigned                       # g_a bookkeeping
    assert sum(ga) == sum(l) == plan.total           # conservation
    if plan.force_count == 0 and not plan.fallback:
        assert max(ga) <= plan.capacity              # capacity (strict, integer cap)
    # weight plan soundness
    W_ = {(e, e // M, d) for e in range(N) for (d, _, _) in plan.chunks[e] if d != e // M}
    assert sorted(W_) == plan.transfers
    if plan.fallback:
        assert plan.transfers == []


def test_golden_traces(golden_dir):
    g = _load(golden_dir, "planner_traces.json")
    for c in g["cases"]:
        p = O1.plan(c["loads"], c["world"], c["alpha"], c["min_chunk"], lam=1.0)
        assert not p.fallback
        assert [[list(ch) for ch in A] for A in p.chunks] == c["chunks"], c["cite"]
        assert p.assigned == c["assigned"], c["cite"]
        assert [list(t) for t in p.transfers] == c["transfers"], c["cite"]
        assert p.force_count == c["force_count"], c["cite"]
        check_invariants(c["loads"], c["world"], c["alpha"], c["min_chunk"], p)


def test_golden_ratios(golden_dir):
    g = _load(golden_dir, "planner_traces.json")["ratios"]
    for c in g["cases"]:
        assert O1.imbalance_ratio(c["loads"]) == pytest.approx(c["ratio"], rel=0, abs=1e-15)
        assert O1.is_balanced(c["loads"], 1.3) == c["balanced_1_3"]


def test_capacity_rounding():
    # (α·S)/P evaluated in float64 and floored once (reading R1); 6.5 -> 6, exact ints stay exact
    assert O1.capacity(13, 2, 1.0) == 6
    assert O1.capacity(1048576, 8, 1.0) == 131072
    assert O1.capacity(10, 3, 1.5) == 5
    assert O1.capacity(0, 4, 2.0) == 0


def test_special_cases():
    # S == 0 -> empty all-native plan, fallback
    p = O1.plan([0, 0, 0, 0], 2)
    assert p.fallback and all(A == [] for A in p.chunks) and p.assigned == [0, 0]
    # P == 1 -> all native even with extreme skew (cap >= S since α >= 1)
    p = O1.plan([100, 0, 3, 0], 1, lam=1.0)
    assert p.chunks == [[(0, 0, 100)], [], [(0, 0, 3)], []] and p.transfers == []
    # uniform loads -> LLA itself is native ("same routing plan as standard EP")
    p = O1.lla([7] * 16, 4, 1.0, 0)
    assert all(A == [(e // 4, 0, 7)] for e, A in enumerate(p.chunks)) and p.transfers == []
    # α·S/P >= max native load -> every expert is Case 1
    l = [9, 1, 2, 8]
    p = O1.lla(l, 2, 2.0, 0)
    assert p.transfers == [] and p.assigned == [10, 10]


def test_validation():
    with pytest.raises(O1.PlannerError):
        O1.plan([1, 2, 3], 2)            # N not divisible by P
    with pytest.raises(O1.PlannerError):
        O1.plan([1, 2], 2, alpha=0.5)
    with pytest.raises(O1.PlannerError):
        O1.plan([1, 2], 2, lam=0.9)
    with pytest.raises(O1.PlannerError):
        O1.plan([1, -2], 2)
    with pytest.raises(O1.PlannerError):
        O1.plan([1, 2], 2, min_chunk=-1)


def test_g120_closed_form():
    """gpt-oss-120b shape, P=8, 32K tokens/rank, K=4, 95 % into 1 expert, λ=1.3, α=1, m=1024
    (P:831-832).  S = P·B·K = 8·cap, so with no force every g_a equals cap exactly; expert 0
    spills to all 7 other devices (|𝒲| = 7); every other expert fits natively."""
    sh = W.CONFIGS["g120"]
    cnt = W.slot_counts(sh.n_experts, sh.tokens_per_rank * sh.top_k, 95, 1)
    l = [int(c) * sh.world for c in cnt]
    p = O1.plan(l, sh.world, 1.0, 1024, 1.3)
    assert not p.fallback and p.force_count == 0
    assert p.capacity == sh.tokens_per_rank * sh.top_k == 131072
    assert p.assigned == [131072] * 8
    assert p.transfers == [(0, 0, d) for d in range(1, 8)]
    assert len(p.chunks[0]) == 8 and all(len(p.chunks[e]) == 1 for e in range(1, 128))
    ep = O1.ep_plan(l, 8)
    # compute-only bound max EP rows / max LLEP rows ("≈7.7" S:441)
    assert 7.6 < max(ep.assigned) / max(p.assigned) < 7.7
    check_invariants(l, 8, 1.0, 1024, p)


def test_balanced_sampled_falls_back():
    """λ=1.3 sends multinomially sampled balanced loads to EP."""
    sh = W.CONFIGS["g120"]
    C = np.stack([np.bincount(W.routing_ids(sh, r, None, 0, sampled=True).ravel(), minlength=128)
                  for r in range(sh.world)])
    l = C.sum(0).tolist()
    assert O1.imbalance_ratio(l) < 1.3
    p = O1.plan(l, 8)
    assert p.fallback and p.transfers == []


def _rand_loads(rng, N, kind):
    if kind == 0:
        return [rng.randint(0, 50) for _ in range(N)]
    if kind == 1:  # skewed: a few hot experts
        l = [rng.randint(0, 20) for _ in range(N)]
        for _ in range(rng.randint(1, 3)):
            l[rng.randrange(N)] += rng.randint(100, 5000)
        return l
    if kind == 2:
        return [rng.choice([0, 0, 1, 3, 1000]) for _ in range(N)]
    return [int(rng.paretovariate(1.2) * 10) for _ in range(N)]


def test_invariant_fuzz():
    """≥10^4 random cases over the SPEC S:610 ranges (N ≤ 512, P ≤ 16, α ∈ [1,3], m ∈ {0,1,64,1024})."""
    rng = random.Random(12345)
    n = 0
    while n < 10000:
        P = rng.choice([1, 2, 3, 4, 8, 16])
        M = rng.choice([1, 2, 3, 4, 8, 16, 32])
        N = P * M
        if N > 512:
            continue
        alpha = rng.choice([1.0, 1.0, 1.25, 1.5, 2.0, rng.uniform(1, 3)])
        m = rng.choice([0, 1, 2, 8, 64, 1024])
        lam = rng.choice([1.0, 1.3, 2.0])
        l = _rand_loads(rng, N, rng.randrange(4))
        p = O1.plan(l, P, alpha, m, lam)
        check_invariants(l, P, alpha, m, p)
        ep = O1.ep_plan(l, P)
        # north star: the max device load is no greater than under EP (empirical, R24)
        assert max(p.assigned) <= max(ep.assigned)
        assert p == O1.plan(l, P, alpha, m, lam)   # determinism
        n += 1


def _argmin_planner(l, P, alpha, m):
    """Independent formulation (the device planner's form): 'first acceptable candidate
    in (g_a+g_p, id) order' == arg-min over acceptable candidates; force == arg-min over all.
    Capacity kept real-valued with a floor per chunk (SPEC S:268 'min(r, floor(avail))')."""
    N = len(l)
    M = N // P
    S = sum(l)
    m_alpha = alpha * S / P
    gp = [sum(l[d * M:(d + 1) * M]) for d in range(P)]
    ga = [0] * P
    chunks = [[] for _ in range(N)]
    forces = 0
    for e in sorted(range(N), key=lambda i: (-l[i], i)):
        if l[e] == 0:
            continue
        ng = e // M
        gp[ng] -= l[e]
        avail = math.floor(m_alpha - ga[ng] - gp[ng])
        r, to = l[e], 0
        if avail >= r:
            chunks[e].append((ng, 0, r)); ga[ng] += r; r = 0
        elif avail >= 1:
            chunks[e].append((ng, 0, avail)); ga[ng] += avail; r -= avail; to = avail
        while r > 0:
            best = None
            for o in range(P):
                if o == ng:
                    continue
                c = min(r, math.floor(m_alpha - ga[o] - gp[o]))
                ok = c >= 1 and not (c < m and r > c)
                key = (ga[o] + gp[o], o)
                if ok and (best is None or key < best[0]):
                    best = (key, o, c)
            if best is None:
                o = min((o for o in range(P) if o != ng), key=lambda o: (ga[o] + gp[o], o))
                c = r
                forces += 1
            else:
                _, o, c = best
            chunks[e].append((o, to, to + c)); ga[o] += c; r -= c; to += c
    return chunks, ga, forces


def test_bruteforce_tiny():
    """All l ∈ {0..7}^N, N ≤ 4, P | N, α ∈ {1, 1.5, 2}, m ∈ {0,1,2,3,8}: invariants, equality with the
    independent arg-min formulation, and the optimum bounds ceil(S/P) ≤ max g_a ≤ EP max."""
    cases = 0
    for N in (1, 2, 3, 4):
        for P in [p for p in (1, 2, 3, 4) if N % p == 0]:
            for l in itertools.product(range(8), repeat=N):
                l = list(l)
                S = sum(l)
                for alpha in (1.0, 1.5, 2.0):
                    for m in (0, 1, 2, 3, 8):
                        p = O1.lla(l, P, alpha, m)
                        check_invariants(l, P, alpha, m, p)
                        ch, ga, forces = _argmin_planner(l, P, alpha, m)
                        assert [list(A) for A in p.chunks] == [list(A) for A in ch], (l, P, alpha, m)
                        assert p.assigned == ga and p.force_count == forces
                        assert -(-S // P) <= max(p.assigned) <= max(O1.ep_plan(l, P).assigned)
                        cases += 1
    assert cases > 20000


def test_bruteforce_exhaustive_optimum():
    """Exhaustive enumeration of every integer split n[e][d] for tiny instances: no assignment beats
    ceil(S/P), and LLA's max load lies between that optimum and EP's (P ∈ {2,3}, N ≤ 3, l_i ≤ 4)."""
    def splits(x, P):
        if P == 1:
            yield (x,)
            return
        for a in range(x + 1):
            for rest in splits(x - a, P - 1):
                yield (a,) + rest
    for P in (2, 3):
        for N in [n for n in (2, 3) if n % P == 0 or n == P]:
            if N % P:
                continue
            for l in itertools.product(range(5), repeat=N):
                opt = None
                for assign in itertools.product(*[list(splits(x, P)) for x in l]):
                    mx = max(sum(a[d] for a in assign) for d in range(P))
                    opt = mx if opt is None else min(opt, mx)
                S = sum(l)
                assert opt == -(-S // P)
                p = O1.lla(list(l), P, 1.0, 0)
                assert opt <= max(p.assigned) <= max(O1.ep_plan(list(l), P).assigned)
