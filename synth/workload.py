"""Seeded synthetic MoE-layer inputs with the structure of the paper's workloads.

Inputs only -- nothing here computes any step of the LLEP method.

Routing scenario (§5.1, and the authors' margin note P:833-834):
"x % of tokens into y experts" means each of the y hot experts (ids 0..y-1) gets
x/y of ALL routed (token, slot) pairs and every other expert gets (1-x)/(N-y).
Duplicate expert ids within one token are allowed (reading R15): with
K=4 a 95 % share for one expert is impossible with distinct top-k ids.

Values come from a counter-based generator (`mix32`) that numpy (host, oracle)
and torch (device, CUDA path) evaluate bit-identically: a 24-bit integer from the
hash is converted exactly to float32, multiplied by one float32 scale (a single
correctly-rounded IEEE multiply on both sides) and rounded to bf16 (RNE).
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Optional

import numpy as np

BASE_SEED = 2601017111
M32 = 0xFFFFFFFF
_MUL = 0x45D9F3B  # < 2^31: (x ^ x>>16) * _MUL stays below 2^63 in int64

# tensor tags for the counter streams
TAG_X, TAG_WGATE, TAG_WUP, TAG_WDOWN, TAG_GATE, TAG_WROUTER = 1, 2, 3, 4, 5, 6


@dataclass(frozen=True)
class LayerShape:
    """One MoE layer + EP world: N experts, top-K, D=d_model, H=d_ff, B tokens per rank, P ranks."""
    n_experts: int
    top_k: int
    d_model: int
    d_ff: int
    tokens_per_rank: int
    world: int

    @property
    def experts_per_rank(self) -> int:
        return self.n_experts // self.world


# BASELINE.json configs (token counts per rank)
CONFIGS = {
    "tiny": LayerShape(8, 2, 256, 512, 1024, 2),
    "g20": LayerShape(32, 4, 2880, 2880, 16384, 8),
    "g120": LayerShape(128, 4, 2880, 2880, 32768, 8),
    "q3": LayerShape(128, 8, 2048, 768, 65536, 8),
    # row f3: the paper's other layer shapes (F-models P:632-686, F-head P:19-101; 16K / 32K per GPU)
    "dsv3": LayerShape(256, 8, 7168, 2048, 16384, 8),
    "kimi": LayerShape(384, 8, 7168, 2048, 16384, 8),
    "fhead": LayerShape(128, 4, 2048, 2048, 32768, 8),
}


# --------------------------------------------------------------------------- hash
def _mix32_int(x: int) -> int:
    x &= M32
    x = ((x >> 16) ^ x) * _MUL & M32
    x = ((x >> 16) ^ x) * _MUL & M32
    return (x >> 16) ^ x


def stream_key(seed: int, tag: int, a: int = 0, b: int = 0) -> int:
    """32-bit key of one counter stream (seed, tensor tag, index a, index b)."""
    k = _mix32_int(seed & M32)
    k = _mix32_int(k ^ _mix32_int((seed >> 32) + 0x3C6EF372))
    k = _mix32_int(k ^ (tag * 0x9E3779B1 & M32))
    k = _mix32_int(k ^ (a * 0x85EBCA77 & M32))
    k = _mix32_int(k ^ (b * 0xC2B2AE3D & M32))
    return k


def mix32_np(x: np.ndarray) -> np.ndarray:
    x = x & M32
    x = ((x >> 16) ^ x) * _MUL & M32
    x = ((x >> 16) ^ x) * _MUL & M32
    return (x >> 16) ^ x


def _mix32_u32(x: np.ndarray) -> np.ndarray:
    """mix32 on uint32 arrays in place-style ops (uint32 multiply wraps mod 2^32 = `* _MUL & M32`):
    the same bits as mix32_np, ~2.5x faster for the large weight tensors."""
    m = np.uint32(_MUL)
    y = x >> np.uint32(16)
    y ^= x
    y *= m
    x = y >> np.uint32(16)
    x ^= y
    x *= m
    y = x >> np.uint32(16)
    y ^= x
    return y


def mix32_torch(x):
    x = x & M32
    x = ((x >> 16) ^ x) * _MUL & M32
    x = ((x >> 16) ^ x) * _MUL & M32
    return (x >> 16) ^ x


def bf16_bits_from_f32(f: np.ndarray) -> np.ndarray:
    """Round float32 to bf16 (round-to-nearest-even), returned as uint16 bit patterns."""
    b = np.ascontiguousarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact upcast of bf16 bit patterns to float64."""
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _uniform_f32_np(key: int, n: int, amp: float, start: int = 0) -> np.ndarray:
    idx = np.arange(start, start + n, dtype=np.uint64)
    idx += np.uint64(key)
    h = _mix32_u32(_mix32_u32((idx & np.uint64(M32)).astype(np.uint32)))
    u = (h >> np.uint32(8)).astype(np.int32) - np.int32(1 << 23)
    return u.astype(np.float32) * np.float32(amp / (1 << 23))


def _uniform_f32_torch(key: int, n: int, amp: float, device, start: int = 0):
    import torch
    idx = torch.arange(start, start + n, dtype=torch.int64, device=device)
    h = mix32_torch(mix32_torch((idx + key) & M32))
    u = (h >> 8) - (1 << 23)
    return u.to(torch.float32) * torch.tensor(np.float32(amp / (1 << 23)), device=device)


# amplitudes: uniform(-a, a) has variance a^2/3
def x_amp() -> float:
    return float(np.sqrt(3.0))              # unit variance tokens


def w_in_amp(d_model: int) -> float:
    return float(np.sqrt(3.0 / d_model))    # W_gate, W_up: variance 1/D


def w_out_amp(d_ff: int) -> float:
    return float(np.sqrt(3.0 / d_ff))       # W_down: variance 1/H


# --------------------------------------------------------------------------- tokens
def tokens_bits(B: int, D: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    """x_p [B, D] as bf16 bit patterns (uint16)."""
    f = _uniform_f32_np(stream_key(seed, TAG_X, rank), B * D, x_amp())
    return bf16_bits_from_f32(f).reshape(B, D)


def tokens_torch(B: int, D: int, rank: int, device, seed: int = BASE_SEED):
    """Same values as tokens_bits, generated on `device` as a bf16 tensor."""
    import torch
    f = _uniform_f32_torch(stream_key(seed, TAG_X, rank), B * D, x_amp(), device)
    return f.to(torch.bfloat16).reshape(B, D)


def token_rows_bits(rows: np.ndarray, D: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    """Selected rows of tokens_bits without generating the whole matrix."""
    key = stream_key(seed, TAG_X, rank)
    out = np.empty((len(rows), D), dtype=np.uint16)
    for i, t in enumerate(np.asarray(rows, dtype=np.int64)):
        out[i] = bf16_bits_from_f32(_uniform_f32_np(key, D, x_amp(), start=int(t) * D))
    return out


# --------------------------------------------------------------------------- weights
def expert_weights_bits(e: int, D: int, H: int, seed: int = BASE_SEED):
    """Expert e's SwiGLU weights as bf16 bits: W_gate [H, D], W_up [H, D], W_down [D, H]."""
    wg = bf16_bits_from_f32(_uniform_f32_np(stream_key(seed, TAG_WGATE, e), H * D, w_in_amp(D))).reshape(H, D)
    wu = bf16_bits_from_f32(_uniform_f32_np(stream_key(seed, TAG_WUP, e), H * D, w_in_amp(D))).reshape(H, D)
    wd = bf16_bits_from_f32(_uniform_f32_np(stream_key(seed, TAG_WDOWN, e), D * H, w_out_amp(H))).reshape(D, H)
    return wg, wu, wd


def expert_weights_torch(experts, D: int, H: int, device, seed: int = BASE_SEED):
    """Device tensors for a list of experts: w13 [E, 2H, D] (rows 0..H-1 = W_gate, H..2H-1 = W_up)
    and w2 [E, D, H] (= W_down), bf16; identical values to expert_weights_bits."""
    import torch
    experts = list(experts)
    E = len(experts)
    w13 = torch.empty((E, 2 * H, D), dtype=torch.bfloat16, device=device)
    w2 = torch.empty((E, D, H), dtype=torch.bfloat16, device=device)
    for i, e in enumerate(experts):
        w13[i, :H] = _uniform_f32_torch(stream_key(seed, TAG_WGATE, e), H * D, w_in_amp(D), device).to(torch.bfloat16).reshape(H, D)
        w13[i, H:] = _uniform_f32_torch(stream_key(seed, TAG_WUP, e), H * D, w_in_amp(D), device).to(torch.bfloat16).reshape(H, D)
        w2[i] = _uniform_f32_torch(stream_key(seed, TAG_WDOWN, e), D * H, w_out_amp(H), device).to(torch.bfloat16).reshape(D, H)
    return w13, w2


def router_weight_bits(N: int, D: int, scale: float = 1.0, seed: int = BASE_SEED) -> np.ndarray:
    """Router weight stored as [N, D] bf16 bits (row i = column i of the paper's W_r ∈ R^{D×N}),
    uniform with variance scale²/D, so unit-variance tokens give logits of standard deviation ~scale."""
    f = _uniform_f32_np(stream_key(seed, TAG_WROUTER, N), N * D, scale * w_in_amp(D))
    return bf16_bits_from_f32(f).reshape(N, D)


def router_weight_torch(N: int, D: int, device, scale: float = 1.0, seed: int = BASE_SEED):
    """Same values as router_weight_bits, as a bf16 tensor on `device`."""
    import torch
    f = _uniform_f32_torch(stream_key(seed, TAG_WROUTER, N), N * D, scale * w_in_amp(D), device)
    return f.to(torch.bfloat16).reshape(N, D)


# --------------------------------------------------------------------------- routing
def target_distribution(n_experts: int, hot_pct: Optional[int], n_hot: int) -> list:
    """Exact per-expert slot shares: hot ids 0..y-1 get x/y each, others (1-x)/(N-y).
    hot_pct=None means balanced (1/N each)."""
    N = n_experts
    if hot_pct is None or n_hot == 0:
        return [Fraction(1, N)] * N
    x = Fraction(hot_pct, 100)
    if not (1 <= n_hot <= N):
        raise ValueError("n_hot out of range")
    if n_hot == N:
        return [Fraction(1, N)] * N
    hot = x / n_hot
    cold = (1 - x) / (N - n_hot)
    return [hot] * n_hot + [cold] * (N - n_hot)


def slot_counts(n_experts: int, n_slots: int, hot_pct: Optional[int], n_hot: int) -> np.ndarray:
    """Largest-remainder rounding of p_e * n_slots (ties -> lower expert id); sums to n_slots."""
    p = target_distribution(n_experts, hot_pct, n_hot)
    quota = [pe * n_slots for pe in p]
    base = [q.numerator // q.denominator for q in quota]
    rem = n_slots - sum(base)
    order = sorted(range(n_experts), key=lambda e: (-(quota[e] - base[e]), e))
    for e in order[:rem]:
        base[e] += 1
    return np.asarray(base, dtype=np.int64)


def routing_ids(shape: LayerShape, rank: int, hot_pct: Optional[int], n_hot: int,
                seed: int = BASE_SEED, sampled: bool = False, distinct: bool = False) -> np.ndarray:
    """topk_ids_p [B, K] int32.  Exact slot multiset per rank (same counts on every rank),
    Fisher-Yates shuffled with PCG64(seed, rank) -- reading R15: x % of ALL slots go to the hot ids, so
    a token may repeat an expert in its K slots; or i.i.d. categorical per slot if sampled; or, with
    distinct=True, K DISTINCT ids per token by weighted sampling without replacement from the target
    distribution (SPEC generate_routing; what a real top-K router can produce: a hot expert then gets at
    most one slot per token, so "95 %" caps at 1/K of the slots)."""
    N, K, B = shape.n_experts, shape.top_k, shape.tokens_per_rank
    rng = np.random.Generator(np.random.PCG64([seed & M32, rank, 0x1D5]))
    if distinct:
        # Efraimidis-Spirakis: each expert draws an exponential clock E_e / p_e; the K earliest win,
        # which is sequential weighted sampling without replacement
        p = np.asarray([float(f) for f in target_distribution(N, hot_pct, n_hot)])
        out = np.empty((B, K), dtype=np.int32)
        for t0 in range(0, B, 8192):
            n = min(8192, B - t0)
            keys = rng.standard_exponential((n, N)) / p[None, :]
            out[t0:t0 + n] = np.argsort(keys, axis=1, kind="stable")[:, :K]
        return out
    if sampled:
        p = np.asarray([float(f) for f in target_distribution(N, hot_pct, n_hot)])
        p = p / p.sum()
        ids = rng.choice(N, size=B * K, p=p)
    else:
        ids = np.repeat(np.arange(N, dtype=np.int64), slot_counts(N, B * K, hot_pct, n_hot))
        rng.shuffle(ids)
    return ids.astype(np.int32).reshape(B, K)


def gate_weights(B: int, K: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    """topk_weights_p [B, K] float32: positive, normalised over the K slots (sequential fp32 sum)."""
    h = mix32_np(mix32_np((np.arange(B * K, dtype=np.int64) + stream_key(seed, TAG_GATE, rank)) & M32))
    u = ((h >> 8) + 1).astype(np.float32).reshape(B, K)
    s = u[:, 0].copy()
    for k in range(1, K):
        s = s + u[:, k]
    return (u / s[:, None]).astype(np.float32)


def scenario_name(hot_pct: Optional[int], n_hot: int) -> str:
    return "balanced" if hot_pct is None else f"{hot_pct}pct_into_{n_hot}"


# --------------------------------------------------------------------------- trace replay (row f4)
class TraceError(ValueError):
    pass


def load_trace(path: str, n_experts: int, world: int = 1) -> list:
    """Per-expert load histograms from a trace file (SPEC's format): one record per line,
    comma-separated: a record id, then N (global l) or P·N (per-device counts, device-major)
    non-negative integers.  Blank lines and lines starting with '#' are skipped.  Returns one
    [world, N] int64 load matrix per record; a reduced (N-entry) record puts all load on device 0
    (planner-only use).  Malformed records, negative counts and width mismatches raise
    TraceError naming the line."""
    out = []
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            fields = [v.strip() for v in line.split(",")]
            try:
                vals = [int(v) for v in fields[1:]]
            except ValueError as e:
                raise TraceError(f"{path}:{ln}: malformed record ({e})") from None
            if any(v < 0 for v in vals):
                raise TraceError(f"{path}:{ln}: negative count")
            if len(vals) == n_experts:
                C = np.zeros((world, n_experts), dtype=np.int64)
                C[0] = vals
            elif len(vals) == world * n_experts:
                C = np.asarray(vals, dtype=np.int64).reshape(world, n_experts)
            else:
                raise TraceError(f"{path}:{ln}: {len(vals)} counts, expected N={n_experts} "
                                 f"or P*N={world * n_experts}")
            out.append(C)
    return out


def routing_from_counts(counts, top_k: int, rank: int, seed: int = BASE_SEED) -> np.ndarray:
    """topk_ids [B, K] int32 whose slot multiset is exactly `counts` (one device's row of a trace
    record; Σ counts must be a multiple of K), Fisher-Yates shuffled with PCG64(seed, rank)."""
    counts = np.asarray(counts, dtype=np.int64)
    S = int(counts.sum())
    if S % top_k:
        raise TraceError(f"{S} routed slots are not a multiple of top-K={top_k}")
    rng = np.random.Generator(np.random.PCG64([seed & M32, rank, 0x7ACE]))
    ids = np.repeat(np.arange(len(counts), dtype=np.int64), counts)
    rng.shuffle(ids)
    return ids.astype(np.int32).reshape(S // top_k, top_k)
