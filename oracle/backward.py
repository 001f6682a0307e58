"""O5 -- backward pass of the MoE layer, float64.  TEST INFRASTRUCTURE (see oracle/__init__).

PAPER.md P:524: "LLEP supports proper gradient propagation.  During the backward pass, the gradients
for the spilled expert weights are returned to their native devices and accumulated with their
native gradients respectively."  The layer is exact, so its gradients are those of Eq. 1
 with SwiGLU experts and the gate on the expert output:

    out[t] = Σ_k w[t,k] · y_tk,   y_tk = W_d a_tk,  a = silu(g) ⊙ u,  g = W_g x_t,  u = W_u x_t

Given the upstream gradient dO[t] = ∂L/∂out[t]:
    dy_tk   = w[t,k] · dO[t]                   dw[t,k] = <y_tk, dO[t]>
    dW_d   += dy_tk ⊗ a_tk                     da      = W_dᵀ dy_tk
    dg      = da ⊙ u ⊙ silu'(g)                du      = da ⊙ silu(g),  silu'(z) = σ(z)(1 + z(1 − σ(z)))
    dW_g   += dg ⊗ x_t      dW_u += du ⊗ x_t   dx[t]  += W_gᵀ dg + W_uᵀ du   (summed in slot order)

`dispatch_combine_backward` executes the same on simulated devices with an LLEP plan: each device
computes partial weight gradients for every expert it ran (native and foreign); foreign partials are
sent to the native device and added there in ascending source-device order.
"""
from __future__ import annotations

from typing import Callable, Dict, Sequence, Tuple

import numpy as np

from . import planner as O1
from . import schedule as O2
from .layer import Weights


def sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def silu(z):
    return z * sigmoid(z)


def dsilu(z):
    s = sigmoid(z)
    return s * (1.0 + z * (1.0 - s))


def expert_backward(X: np.ndarray, dY: np.ndarray, w: Weights):
    """One expert on rows X [n, D] with output gradients dY [n, D] (gate already applied).
    Returns (dX [n, D], y [n, D], (dW_g [H, D], dW_u [H, D], dW_d [D, H]))."""
    wg, wu, wd = w
    g = X @ wg.T
    u = X @ wu.T
    a = silu(g) * u
    y = a @ wd.T
    dWd = dY.T @ a
    da = dY @ wd
    dg = da * u * dsilu(g)
    du = da * silu(g)
    dWg = dg.T @ X
    dWu = du.T @ X
    dX = dg @ wg + du @ wu
    return dX, y, (dWg, dWu, dWd)


def moe_backward(x: np.ndarray, ids: np.ndarray, gates: np.ndarray, dout: np.ndarray,
                 weights: Callable[[int], Weights]):
    """Gradients of L = Σ_t <out[t], dout[t]> for one rank's tokens (dense definition).
    Returns dx [T, D], dgates [T, K], dW {e: (dW_g, dW_u, dW_d)} for every routed expert."""
    x = np.asarray(x, dtype=np.float64)
    dout = np.asarray(dout, dtype=np.float64)
    gates = np.asarray(gates, dtype=np.float64)
    T, K = ids.shape
    D = x.shape[1]
    dX_slot = np.zeros((T, K, D))
    dgates = np.zeros((T, K))
    dW: Dict[int, Tuple[np.ndarray, np.ndarray, np.ndarray]] = {}
    for e in np.unique(ids):
        tt, kk = np.nonzero(ids == e)
        dY = gates[tt, kk, None] * dout[tt]
        dX, y, dw = expert_backward(x[tt], dY, weights(int(e)))
        dX_slot[tt, kk] = dX
        dgates[tt, kk] = np.einsum("nd,nd->n", y, dout[tt])
        dW[int(e)] = dw
    dx = np.zeros((T, D))
    for k in range(K):  # slot order
        dx += dX_slot[:, k]
    return dx, dgates, dW


def dispatch_combine_backward(x: Sequence[np.ndarray], ids: Sequence[np.ndarray],
                              gates: Sequence[np.ndarray], dout: Sequence[np.ndarray],
                              weights: Callable[[int], Weights], n_experts: int, world: int,
                              mode: str = "llep", alpha: float = 1.0, min_chunk: int = 1024,
                              lam: float = 1.3):
    """Backward on simulated devices under the EP / LLEP plan of the forward (Alg. 4 + P:524).
    Returns (dx per rank, dgates per rank, dW per expert on its native device, plan)."""
    P, N = world, n_experts
    M = N // P
    C = O2.load_matrix(ids, N)
    l = C.sum(axis=0)
    plan = O1.ep_plan(l, P, alpha, fallback=False) if mode == "ep" else O1.plan(l, P, alpha, min_chunk, lam)
    # rows each device receives: (expert) -> list of (pos, src rank, flat slot)
    recv = [dict() for _ in range(P)]
    for p in range(P):
        flat = np.asarray(ids[p]).reshape(-1)
        dev, pos = O2.slot_destinations(plan, C, flat, p)
        for j in range(flat.size):
            recv[int(dev[j])].setdefault(int(flat[j]), []).append((int(pos[j]), p, j))
    dX_slot = [np.zeros((np.asarray(i).shape[0], np.asarray(i).shape[1], x[0].shape[1])) for i in ids]
    dg_slot = [np.zeros(np.asarray(i).shape) for i in ids]
    partial: Dict[Tuple[int, int], Tuple[np.ndarray, np.ndarray, np.ndarray]] = {}
    for d in range(P):
        for e, rows in recv[d].items():
            rows.sort()
            K = [np.asarray(ids[p]).shape[1] for p in range(P)]
            X = np.stack([x[p][j // K[p]] for (_, p, j) in rows])
            dY = np.stack([np.asarray(gates[p]).reshape(-1)[j] * dout[p][j // K[p]] for (_, p, j) in rows])
            dX, y, dw = expert_backward(X, dY, weights(e))
            for (_, p, j), dxr, yr in zip(rows, dX, y):
                dX_slot[p][j // K[p], j % K[p]] = dxr
                dg_slot[p][j // K[p], j % K[p]] = float(yr @ dout[p][j // K[p]])
            partial[(e, d)] = dw
    # foreign partials return to the native device, summed in ascending device order
    dW = {}
    for e in range(N):
        ng = O1.native_device(e, M)
        devs = sorted(d for (ee, d) in partial if ee == e)
        if not devs:
            continue
        acc = None
        for d in ([ng] if ng in devs else []) + [d for d in devs if d != ng]:
            pw = partial[(e, d)]
            acc = [a.copy() for a in pw] if acc is None else [a + b for a, b in zip(acc, pw)]
        dW[e] = tuple(acc)
    dx = []
    for p in range(P):
        o = np.zeros((dX_slot[p].shape[0], dX_slot[p].shape[2]))
        for k in range(dX_slot[p].shape[1]):
            o += dX_slot[p][:, k]
        dx.append(o)
    return dx, dg_slot, dW, plan
