"""O2 -- load matrix, stable re-indexing and per-slot destinations.  TEST INFRASTRUCTURE.

PAPER.md:
  P:537      l <- "sum of loads of global experts across all GPUs"; we keep the
             all-gathered [P, N] matrix C (l = column sums) because the global ->
             local offset mapping needs per-source counts (reading R26).
  P:282      re-indexing: per-expert batches formed by a STABLE sort of the flat
             (token, slot) list ([a,b,c,d] -> experts [2,6,2,1] -> [d,a,c,b]).
  P:299-303  sort(flatten(I_p)), index_select, slice.
  P:547-548  "build chunks of B̄_p from 𝒜": a chunk (d, s, t) of expert e covers
             global positions [s, t) of e's token range.

Reading R11 (paper silent): expert e's global token order is rank-major -- all of
rank 0's slots routed to e in flat order t*K+k, then rank 1's, and so on.
Reading R11' (round 2, the CUDA path's default; also paper-silent): the same per-source blocks in
flat order, but for an expert with MORE than one chunk the blocks follow the devices of its chunks in
plan order (first appearance), then the remaining ranks ascending -- "chunk-aligned": a spill device's
chunk then holds its own rows wherever the counts allow, so they need no transfer.  Experts with at
most one chunk keep R11.  Both orders cover every slot exactly once; which one a call uses is a
context setting (llep_context_set_token_order).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np

from .planner import Plan, native_device


def local_counts(ids: np.ndarray, n_experts: int) -> np.ndarray:
    """cnt_p[e] = #{(t,k): ids[t,k] = e}  (one row of the load matrix)."""
    flat = np.asarray(ids).reshape(-1)
    if flat.size and (flat.min() < 0 or flat.max() >= n_experts):
        raise ValueError("routing index out of range")
    return np.bincount(flat, minlength=n_experts).astype(np.int64)


def load_matrix(ids_per_rank: Sequence[np.ndarray], n_experts: int) -> np.ndarray:
    """C [P, N]: row p = rank p's per-expert slot counts (the all-gathered statistic)."""
    return np.stack([local_counts(ids, n_experts) for ids in ids_per_rank])


def stable_reindex(ids: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """P:282 / P:299: stable sort of the flattened slots by expert.
    Returns (perm, sorted_ids): perm[i] = flat slot at sorted position i."""
    flat = np.asarray(ids).reshape(-1)
    perm = np.argsort(flat, kind="stable")
    return perm, flat[perm]


def local_rank_in_expert(ids: np.ndarray) -> np.ndarray:
    """r_j = #{j' < j : ids[j'] = ids[j]} for every flat slot j (position inside the
    rank's own per-expert batch B_i of P:282): in the stable sorted order, a slot's rank is its
    sorted position minus the sorted position of the first slot of its expert."""
    flat = np.asarray(ids).reshape(-1)
    perm, sorted_ids = stable_reindex(flat)
    first = np.searchsorted(sorted_ids, sorted_ids, side="left")   # start of each slot's expert run
    r = np.empty(flat.size, dtype=np.int64)
    r[perm] = np.arange(flat.size) - first
    return r


def source_order(plan: Plan, e: int) -> List[int]:
    """R11' order of the sources' blocks in expert e's global range: e's chunk devices in plan order
    (first appearance), then the other ranks ascending; rank-major (R11) when e has <= 1 chunk."""
    P = plan.world
    A = plan.chunks[e]
    if len(A) <= 1:
        return list(range(P))
    order: List[int] = []
    for (d, _s, _t) in A:
        if d not in order:
            order.append(d)
    return order + [q for q in range(P) if q not in order]


def global_index(ids: np.ndarray, C: np.ndarray, rank: int, plan: Plan = None) -> np.ndarray:
    """gidx_j = (slots of e from the sources before p) + r_j.  plan=None: rank-major, the sources
    before p are q < p (R11); with a plan: the sources before p in source_order(plan, e) (R11')."""
    flat = np.asarray(ids).reshape(-1)
    if plan is None:
        base = C[:rank].sum(axis=0) if rank > 0 else np.zeros(C.shape[1], dtype=np.int64)
    else:
        base = np.zeros(C.shape[1], dtype=np.int64)
        for e in range(C.shape[1]):
            order = source_order(plan, e)
            base[e] = sum(int(C[q][e]) for q in order[:order.index(rank)])
    return base[flat] + local_rank_in_expert(flat)


def chunk_of(plan: Plan, e: int, g: int) -> Tuple[int, int]:
    """(chunk ordinal, device) of the unique chunk of expert e with start <= g < end."""
    for ci, (d, s, t) in enumerate(plan.chunks[e]):
        if s <= g < t:
            return ci, d
    raise ValueError(f"global index {g} of expert {e} not covered by the plan")


def rows_on_device(plan: Plan, e: int, d: int) -> int:
    return sum(t - s for (dd, s, t) in plan.chunks[e] if dd == d)


def slot_destinations(plan: Plan, C: np.ndarray, ids: np.ndarray, rank: int,
                      aligned: bool = False) -> Tuple[np.ndarray, np.ndarray]:
    """For each flat slot j of rank p: destination device d_j (the device of the unique chunk of
    expert e_j with start <= gidx_j < end) and the slot's position among expert e_j's
    rows on d_j (the chunks of e on d concatenated in plan order: the chunk's offset among them
    plus gidx_j - start).  aligned: global index in the R11' order instead of R11."""
    flat = np.asarray(ids).reshape(-1)
    g = global_index(flat, C, rank, plan if aligned else None)
    dev = np.full(flat.size, -1, dtype=np.int64)
    pos = np.empty(flat.size, dtype=np.int64)
    for e in np.unique(flat):
        of_e = flat == e
        off_on = {}                                   # rows of e's earlier chunks on each device
        for (d0, s, t) in plan.chunks[int(e)]:
            base = off_on.get(d0, 0)
            hit = of_e & (g >= s) & (g < t)
            dev[hit] = d0
            pos[hit] = base + (g[hit] - s)
            off_on[d0] = base + (t - s)
    if flat.size and (dev < 0).any():
        raise ValueError("uncovered slot")
    return dev, pos


def send_schedule(plan: Plan, C: np.ndarray) -> Dict[Tuple[int, int], List[Tuple[int, int, int]]]:
    """SPEC materialize_send_schedule: for source p and expert e, the list of
    (dst, local_start, local_end) slices of p's local rows of e, intersecting every plan chunk
    with p's sub-range [Σ_{q<p} C[q][e], Σ_{q<=p} C[q][e]) of e's global range."""
    P, N = C.shape
    if [sum(t - s for (_, s, t) in plan.chunks[e]) for e in range(N)] != list(C.sum(axis=0)):
        raise ValueError("plan/load inconsistency")
    out: Dict[Tuple[int, int], List[Tuple[int, int, int]]] = {}
    for e in range(N):
        lo = 0
        for p in range(P):
            hi = lo + int(C[p][e])
            sl = []
            for (d, s, t) in plan.chunks[e]:
                a, b = max(s, lo), min(t, hi)
                if a < b:
                    sl.append((d, a - lo, b - lo))
            out[(p, e)] = sl
            lo = hi
    return out


def foreign_sets(plan: Plan) -> List[List[int]]:
    """S_d: experts device d computes but does not host (Alg. 4)."""
    M = plan.experts_per_device
    S: List[set] = [set() for _ in range(plan.world)]
    for e, A in enumerate(plan.chunks):
        for (d, _s, _t) in A:
            if d != native_device(e, M):
                S[d].add(e)
    return [sorted(s) for s in S]


def device_rows(plan: Plan) -> List[int]:
    """R_d = rows device d computes = g_a[d] (recomputed from the chunks)."""
    R = [0] * plan.world
    for A in plan.chunks:
        for (d, s, t) in A:
            R[d] += t - s
    return R
