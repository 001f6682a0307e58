"""Shared helpers for the GPU layer parity tests: seeded inputs (synth) for one rank, the CUDA
path through the C ABI, and the float64 oracle reference for the same inputs."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from synth import workload as W  # noqa: E402

TOL_MAX_REL = 2e-2   # north star: max relative error (reading R21)
TOL_REL_L2 = 5e-3    # north star: relative L2 error


def rank_inputs(shape: W.LayerShape, rank: int, hot_pct, n_hot: int, seed: int, device, sampled=False):
    import torch
    B, K, D, H, M = shape.tokens_per_rank, shape.top_k, shape.d_model, shape.d_ff, shape.experts_per_rank
    ids = W.routing_ids(shape, rank, hot_pct, n_hot, seed, sampled=sampled)
    gates = W.gate_weights(B, K, rank, seed)
    x = W.tokens_torch(B, D, rank, device, seed)
    w13, w2 = W.expert_weights_torch(range(rank * M, (rank + 1) * M), D, H, device, seed)
    return (x, torch.from_numpy(ids).to(device), torch.from_numpy(gates).to(device), w13, w2, ids, gates)


class OracleWeights:
    """float64 expert weights (exact bf16 values) generated on demand by the synth generator."""

    def __init__(self, D: int, H: int, seed: int):
        self.D, self.H, self.seed = D, H, seed
        self.cache = {}

    def __call__(self, e: int):
        if e not in self.cache:
            wg, wu, wd = W.expert_weights_bits(e, self.D, self.H, self.seed)
            self.cache[e] = (W.bf16_bits_to_f64(wg), W.bf16_bits_to_f64(wu), W.bf16_bits_to_f64(wd))
        return self.cache[e]


def oracle_rank_output(shape: W.LayerShape, rank: int, ids: np.ndarray, gates: np.ndarray, seed: int,
                       rows=None, weights=None):
    """O3 for (a subset of) one rank's tokens."""
    from oracle import layer as O3
    D, H = shape.d_model, shape.d_ff
    if rows is None:
        rows = np.arange(ids.shape[0])
    xb = W.token_rows_bits(rows, D, rank, seed) if len(rows) < ids.shape[0] else W.tokens_bits(ids.shape[0], D, rank, seed)
    x = W.bf16_bits_to_f64(xb)
    weights = weights or OracleWeights(D, H, seed)
    return O3.moe_forward(x, ids[rows], gates[rows].astype(np.float64), weights)


def errors(y: np.ndarray, r: np.ndarray):
    from oracle import layer as O3
    return O3.relative_errors(y, r)
