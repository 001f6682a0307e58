"""O3 -- the MoE layer output by its plain definition, float64.  TEST INFRASTRUCTURE.

LLEP is exact: its output is the MoE output of Eq. 1,
    h = Σ_i g_i FFN_i(u),
whatever the plan.  Experts are SwiGLU modules with three weight matrices:
    FFN_e(u) = W_down,e ( silu(W_gate,e u) ⊙ (W_up,e u) ),  silu(z) = z / (1 + e^-z)
and the gate multiplies the expert OUTPUT (Ĥ_i = Ĝ_i ⊙ B̂_i W_i, P:307 / P:554).
Slots are summed per token in slot order k = 0..K-1 (Alg. 1 "sum(H_p, dim=K)").

Inputs are the exact bf16 values of x and W upcast to float64, and the fp32 gates
upcast -- no bf16 rounding is modelled (reading R18).  `linear` mode evaluates Eq. 1's
simple form FFN_i(u) = uᵀW_i for the textbook pins.
"""
from __future__ import annotations

from typing import Callable, Tuple

import numpy as np

Weights = Tuple[np.ndarray, np.ndarray, np.ndarray]  # W_gate [H,D], W_up [H,D], W_down [D,H] float64


def silu(z: np.ndarray) -> np.ndarray:
    return z / (1.0 + np.exp(-z))


def swiglu_ffn(u: np.ndarray, w: Weights) -> np.ndarray:
    """FFN_e(u) for the rows of u [n, D] -> [n, D]."""
    wg, wu, wd = w
    return (silu(u @ wg.T) * (u @ wu.T)) @ wd.T


def moe_forward(x: np.ndarray, ids: np.ndarray, gates: np.ndarray,
                weights: Callable[[int], Weights], row_chunk: int = 65536) -> np.ndarray:
    """Eq. 1 for every token of one rank: out[t] = Σ_k gates[t,k] · FFN_{ids[t,k]}(x[t]).

    x [T, D] float64, ids [T, K] int, gates [T, K] float64 -> out [T, D] float64.
    Rows of each expert are processed in chunks of `row_chunk` to bound host memory.
    """
    x = np.asarray(x, dtype=np.float64)
    ids = np.asarray(ids)
    gates = np.asarray(gates, dtype=np.float64)
    T, K = ids.shape
    D = x.shape[1]
    Y = np.zeros((T, K, D), dtype=np.float64)          # FFN output per (token, slot)
    for e in np.unique(ids):
        w = weights(int(e))
        tt, kk = np.nonzero(ids == e)
        for a in range(0, tt.size, row_chunk):
            t_, k_ = tt[a:a + row_chunk], kk[a:a + row_chunk]
            Y[t_, k_] = swiglu_ffn(x[t_], w)
    out = np.zeros((T, D), dtype=np.float64)
    for k in range(K):                                 # slot order
        out += gates[:, k, None] * Y[:, k]
    return out


def moe_forward_linear(x: np.ndarray, ids: np.ndarray, gates: np.ndarray,
                       W: Callable[[int], np.ndarray]) -> np.ndarray:
    """Eq. 1 with FFN_i(u) = uᵀ W_i, W_i [D, H]."""
    x = np.asarray(x, dtype=np.float64)
    T, K = ids.shape
    H = W(int(ids.reshape(-1)[0])).shape[1] if ids.size else 0
    out = np.zeros((T, H), dtype=np.float64)
    for k in range(K):
        for t in range(T):
            out[t] += gates[t, k] * (x[t] @ W(int(ids[t, k])))
    return out


def relative_errors(y: np.ndarray, r: np.ndarray) -> Tuple[float, float]:
    """(max_rel, rel_L2) as the north star's tolerance is read (R21):
    max|y-r| / max|r|  and  ||y-r||_2 / ||r||_2 over the whole output."""
    y = np.asarray(y, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    diff = y - r
    mr = float(np.abs(diff).max() / max(np.abs(r).max(), 1e-300)) if r.size else 0.0
    l2 = float(np.linalg.norm(diff) / max(np.linalg.norm(r), 1e-300)) if r.size else 0.0
    return mr, l2
