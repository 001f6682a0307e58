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


def config_shape(cfg: str) -> W.LayerShape:
    """A synth.CONFIGS name, or "shape:N,K,D,H,B" for a test-only layer shape (world size set by the caller)."""
    if cfg.startswith("shape:"):
        n, k, d, h, b = (int(v) for v in cfg[len("shape:"):].split(","))
        return W.LayerShape(n, k, d, h, b, 1)
    return W.CONFIGS[cfg]


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

    def prefetch(self, experts, threads: int = 0):
        """Generate the weights of many experts in parallel (numpy releases the GIL in its ufuncs)."""
        from concurrent.futures import ThreadPoolExecutor
        todo = sorted({int(e) for e in experts} - set(self.cache))
        if not todo:
            return
        n = threads or min(32, os.cpu_count() or 1)
        with ThreadPoolExecutor(max_workers=n) as ex:
            for e, w in zip(todo, ex.map(self._make, todo)):
                self.cache[e] = w

    def _make(self, e: int):
        wg, wu, wd = W.expert_weights_bits(e, self.D, self.H, self.seed)
        return (W.bf16_bits_to_f64(wg), W.bf16_bits_to_f64(wu), W.bf16_bits_to_f64(wd))

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
    if hasattr(weights, "prefetch"):
        weights.prefetch(np.unique(ids[rows]))
    return O3.moe_forward(x, ids[rows], gates[rows].astype(np.float64), weights)


def errors(y: np.ndarray, r: np.ndarray):
    from oracle import layer as O3
    return O3.relative_errors(y, r)


def expected_layout(plan, d: int, row_align: int = 256):
    """Device d's group table as rows a5 of SURVEY §8 define it, derived here from the oracle plan:
    native experts of d with rows on d (ascending id), then the foreign experts S_d (ascending id); each
    group holds e's chunks on d concatenated in plan order and starts at the running sum of the earlier
    groups' row counts rounded up to `row_align` (the GEMM's M tile).  -> [(expert, wslot, base, n)]"""
    from oracle import schedule as O2
    M = plan.experts_per_device
    out, base, f = [], 0, 0
    for native in (True, False):
        for e in range(plan.n_experts):
            if (e // M == d) != native:
                continue
            n = O2.rows_on_device(plan, e, d)
            if n == 0:
                continue
            out.append((e, e - d * M if native else -1 - f, base, n))
            f += 0 if native else 1
            base += -(-n // row_align) * row_align
    return out


def check_index_work(res, key: str, plan, ids_all, n_experts: int, aligned: bool = None):
    """Rows a1-a5 bit-exact against O2 on every rank (north star: integer / index work bit-exact):
    the all-gathered load matrix C, every slot's stable local rank r_j, every device's group table,
    and every slot's destination (device, row) = (d_j, base_d[e_j] + pos_j) with (d_j, pos_j) from
    O2.slot_destinations (global index in the context's token order -- chunk-aligned R11' by default,
    rank-major R11 when LLEP_TEST_ORDER=rank_major -- and the chunk lookup of P:547-548)."""
    if aligned is None:
        aligned = os.environ.get("LLEP_TEST_ORDER", "chunk_aligned") != "rank_major"
    from oracle import schedule as O2
    P = len(ids_all)
    C = O2.load_matrix(ids_all, n_experts)
    base = []
    for d in range(P):
        lay = expected_layout(plan, d)
        g = res[d][f"{key}_groups"]
        got = [tuple(int(v) for v in row[:4]) for row in g]
        assert got == lay, (key, d, got[:4], lay[:4])
        base.append({e: b for (e, _w, b, _n) in lay})
    for p in range(P):
        assert np.array_equal(res[p][f"{key}_lm"], C), (key, p)
        assert np.array_equal(res[p][f"{key}_lr"], O2.local_rank_in_expert(ids_all[p])), (key, p)
        dev, pos = O2.slot_destinations(plan, C, ids_all[p], p, aligned=aligned)
        flat = ids_all[p].reshape(-1)
        row = np.array([base[d][int(e)] for d, e in zip(dev, flat)], dtype=np.int64) + pos
        dst = res[p][f"{key}_dst"]
        assert np.array_equal(dst[:, 0], dev), (key, p)
        assert np.array_equal(dst[:, 1], row), (key, p)


def boundary_tokens(plan, ids_all, n_experts: int, extra: int = 16):
    """Per rank, the tokens whose slots sit at the first and last global index of every plan chunk (so
    every chunk and group boundary on every device is sampled), plus each rank's first `extra` tokens.
    -> {rank: sorted token indices}."""
    from oracle import schedule as O2
    P = len(ids_all)
    C = O2.load_matrix(ids_all, n_experts)
    K = ids_all[0].shape[1]
    gidx = [O2.global_index(ids_all[p], C, p, plan) for p in range(P)]   # chunk-aligned order (R11')
    flat = [ids_all[p].reshape(-1) for p in range(P)]
    want = {p: set(range(min(extra, ids_all[p].shape[0]))) for p in range(P)}
    for e, A in enumerate(plan.chunks):
        for (_d, s, t) in A:
            for g in (s, t - 1):
                for p in range(P):
                    hit = np.nonzero((flat[p] == e) & (gidx[p] == g))[0]
                    if hit.size:
                        want[p].add(int(hit[0]) // K)
                        break
    return {p: np.array(sorted(v), dtype=np.int64) for p, v in want.items()}
