"""O6 -- the router of Eq. 2, float64.  TEST INFRASTRUCTURE (see oracle/__init__).

PAPER.md §2.1, Eq. 2: for a token u ∈ R^D and the router weight W_r ∈ R^{D×N},
    s_i = softmax_i(uᵀ W_r),
    g_i = s_i if s_i ∈ top-K({s_j | 0 ≤ j ≤ N-1}, K) else 0,
and h = Σ_i g_i FFN_i(u) (Eq. 1).  The gate of a selected expert is its softmax probability over
ALL N experts (no renormalisation over the K selected -- the paper writes none).

Readings (R31-R33):
  R31 the K selected slots are listed in descending s, ties broken by the lower expert id (the paper
      does not order the K slots; the order fixes the slot index k that Eq. 1's K-sum runs over);
  R32 ties in the top-K membership itself are broken the same way (lower id wins);
  R33 W_r is stored as its transpose [N, D] (one row per expert, like the expert weights) by the
      CUDA path; this oracle takes the paper's W_r [D, N].
"""
from __future__ import annotations

import numpy as np


def logits(x: np.ndarray, w_r: np.ndarray) -> np.ndarray:
    """z[t, i] = x[t]ᵀ W_r[:, i], x [T, D], W_r [D, N] -> [T, N] float64."""
    return np.asarray(x, dtype=np.float64) @ np.asarray(w_r, dtype=np.float64)


def softmax(z: np.ndarray) -> np.ndarray:
    """s_i = exp(z_i) / Σ_j exp(z_j) per row; written with the row max subtracted from
    every exponent, which leaves the quotient unchanged and keeps exp finite."""
    z = np.asarray(z, dtype=np.float64)
    e = np.exp(z - z.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def top_k(s: np.ndarray, K: int) -> np.ndarray:
    """Indices of the K largest entries of the vector s, largest first, ties -> lower index
    (R31, R32): K rounds of "take the first maximum among the not yet taken"."""
    s = np.asarray(s, dtype=np.float64)
    taken = np.zeros(s.shape[0], dtype=bool)
    out = []
    for _ in range(K):
        best = -1
        for i in range(s.shape[0]):
            if not taken[i] and (best < 0 or s[i] > s[best]):
                best = i
        taken[best] = True
        out.append(best)
    return np.asarray(out, dtype=np.int64)


def route_from_logits(z: np.ndarray, K: int):
    """Eq. 2 from given logits z [T, N]: (ids [T, K] int64, gates [T, K] float64).
    Selection on s = softmax(z) (monotone in z, so it equals selection on z)."""
    s = softmax(z)
    ids = np.stack([top_k(row, K) for row in s]) if len(s) else np.zeros((0, K), dtype=np.int64)
    gates = np.take_along_axis(s, ids, axis=1) if len(s) else np.zeros((0, K))
    return ids, gates


def route(x: np.ndarray, w_r: np.ndarray, K: int):
    """The router of Eq. 2 for the tokens x [T, D]: (ids [T, K], gates [T, K], logits [T, N])."""
    z = logits(x, w_r)
    ids, gates = route_from_logits(z, K)
    return ids, gates, z


def dense_gates(ids: np.ndarray, gates: np.ndarray, n_experts: int) -> np.ndarray:
    """Eq. 2's g vector per token (N entries, zero off the top-K) from the sparse (ids, gates)."""
    T = ids.shape[0]
    g = np.zeros((T, n_experts))
    for t in range(T):
        for k in range(ids.shape[1]):
            g[t, ids[t, k]] += gates[t, k]
    return g
