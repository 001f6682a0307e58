"""O4 -- standard EP (Alg. 1) and LLEP (Alg. 4) executed on simulated devices.  TEST INFRASTRUCTURE.

Each simulated device p holds its tokens, gates and ids and its native experts
[pM, (p+1)M).  The steps follow Alg. 4 in order:
  P:537       l from the all-gathered load matrix C
  P:538-541   λ test -> Alg. 1 (the all-native plan)
  P:542-544   stable sort + index_select of the flat slots
  P:546       𝒜, 𝒲 <- LLA(l, M)
  P:547-551   chunks per destination, All-to-All of tokens and gates
  P:552       P2P transfer of W_j, j ∈ S
  P:554       Ĥ_i = Ĝ_i ⊙ B̂_i W_i for native and foreign experts
  P:556-561   reverse All-to-All, reverse sort, reshape (B_p, K, ·), sum over K
The result must equal O3 (layer.moe_forward) -- LLEP is exact.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence, Tuple

import numpy as np

from . import planner as O1
from . import schedule as O2
from .layer import Weights, swiglu_ffn


def dispatch_combine(x: Sequence[np.ndarray], ids: Sequence[np.ndarray], gates: Sequence[np.ndarray],
                     weights: Callable[[int], Weights], n_experts: int, world: int,
                     mode: str = "llep", alpha: float = 1.0, min_chunk: int = 1024, lam: float = 1.3):
    """Simulate one layer step on `world` devices.  mode = 'ep' (Alg. 1) or 'llep' (Alg. 4).
    Returns (outputs per device [B_p, D] float64, plan, stats)."""
    P, N = world, n_experts
    M = N // P
    C = O2.load_matrix(ids, N)
    l = C.sum(axis=0)
    if mode == "ep":
        plan = O1.ep_plan(l, P, alpha, fallback=False)
    else:
        plan = O1.plan(l, P, alpha, min_chunk, lam)
    # devices' receive buffers: dev -> expert -> list of (src rank, flat slot, row, gate)
    recv: List[Dict[int, List[Tuple[int, int, np.ndarray, float]]]] = [dict() for _ in range(P)]
    for p in range(P):
        flat_ids = np.asarray(ids[p]).reshape(-1)
        K = np.asarray(ids[p]).shape[1]
        dev, pos = O2.slot_destinations(plan, C, flat_ids, p)
        for j in range(flat_ids.size):                               # P:550-551 All-to-All
            e = int(flat_ids[j])
            recv[int(dev[j])].setdefault(e, []).append(
                (int(pos[j]), p, j, x[p][j // K], float(np.asarray(gates[p]).reshape(-1)[j])))
    # P2P weight import: a device may compute e iff native or (e, native, d) ∈ 𝒲
    imported = {(e, d) for (e, _s, d) in plan.transfers}
    results: List[Dict[Tuple[int, int], np.ndarray]] = [dict() for _ in range(P)]
    for d in range(P):
        for e, rows in recv[d].items():
            if O1.native_device(e, M) != d and (e, d) not in imported:
                raise AssertionError(f"device {d} computes expert {e} without its weights")
            rows.sort(key=lambda r: r[0])                            # position order on d
            if [r[0] for r in rows] != list(range(len(rows))):
                raise AssertionError("positions on a device are not a permutation")
            B_hat = np.stack([r[3] for r in rows])
            G_hat = np.asarray([r[4] for r in rows])
            H_hat = G_hat[:, None] * swiglu_ffn(B_hat, weights(e))
            for r, h in zip(rows, H_hat):
                results[r[1]][(r[2],)] = h                           # P:556 reverse All-to-All
    outs = []
    for p in range(P):
        B, K = np.asarray(ids[p]).shape
        D = x[p].shape[1]
        Hs = np.zeros((B, K, D))
        for (j,), h in results[p].items():                           # P:559-560 reverse sort, reshape
            Hs[j // K, j % K] = h
        out = np.zeros((B, D))
        for k in range(K):                                           # P:561 sum over K, slot order
            out += Hs[:, k]
        outs.append(out)
    stats = {
        "device_rows": O2.device_rows(plan),
        "foreign": O2.foreign_sets(plan),
        "n_transfers": len(plan.transfers),
    }
    return outs, plan, stats
