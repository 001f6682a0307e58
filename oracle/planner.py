"""O1 -- the LLEP planner, step by step in the paper's order.  TEST INFRASTRUCTURE (see oracle/__init__).

Follows PAPER.md:
  Alg. 4 head   P:537-541   l <- global loads; if max(l)/mean(l) < λ -> standard EP
  Alg. 2 (LLA)  P:382-423   sort loads descending, per expert Case 1 / 2 / 3
  Alg. 3 (LLAS) P:486-513   least-loaded spill with the "chunk too small" skip and force-assign
  𝒲             P:420, P:522  (expert, native -> dst) for every non-native chunk

Readings of silent / ambiguous points:
  R1  m_α = α·Σl/P is evaluated as float64 (α·S)/P and floored once: cap.
      All later comparisons are exact integer arithmetic (chunks are token counts).
  R2  Case 2 needs integer na > 0 (0 < m_α-g_a-g_p < 1 -> Case 3, no empty native chunk).
  R3  LLAS skips a candidate whose chunk c <= 0 (P:494-497 silent; otherwise m=0 livelocks).
  R4  "skip" = try the next candidate in the sorted order; the first acceptable wins.
  R5  ties: experts by (load desc, id asc); devices by (g_a+g_p asc, id asc).
  R6  zero-load experts get no chunk and no transfer.
  R7  force-assign puts the whole remainder on o[0], ignoring m and the capacity.
  R8  the native chunk of Case 2 is exempt from m (P:406-411 applies no m test).
  R9  λ test: strict <, mean over all N experts, ratio = max/(S/N) in float64; S=0 -> balanced.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

Chunk = Tuple[int, int, int]  # (device, start, end) over the expert's global token range


class PlannerError(ValueError):
    pass


@dataclass
class Plan:
    n_experts: int
    world: int
    chunks: List[List[Chunk]]          # 𝒜: per expert, in the order LLA/LLAS appended them
    assigned: List[int]                # g_a per device
    capacity: int                      # floor(m_α)
    total: int                         # S = Σ l
    fallback: bool                     # True iff the λ test (or S == 0) selected standard EP
    force_count: int = 0               # number of LLAS force-assigns
    transfers: List[Tuple[int, int, int]] = field(default_factory=list)  # 𝒲: (expert, src, dst) sorted

    @property
    def experts_per_device(self) -> int:
        return self.n_experts // self.world


def validate(loads: Sequence[int], world: int, alpha: float, min_chunk: int, lam: float) -> None:
    N = len(loads)
    if world < 1 or N < 1 or N % world != 0:
        raise PlannerError("N not divisible by P")
    if not (alpha >= 1.0):
        raise PlannerError("alpha < 1")
    if not (lam >= 1.0):
        raise PlannerError("lambda < 1")
    if min_chunk < 0:
        raise PlannerError("min_chunk < 0")
    if any(int(x) < 0 for x in loads):
        raise PlannerError("negative load")


def native_device(e: int, M: int) -> int:
    """ng <- floor(i / M)  (Alg. 2)."""
    return e // M


def imbalance_ratio(loads: Sequence[int]) -> float:
    """max(l) / mean(l)  (Alg. 4); 1.0 for an empty batch (R9)."""
    S = sum(int(x) for x in loads)
    if S == 0:
        return 1.0
    return float(max(int(x) for x in loads)) / (float(S) / float(len(loads)))


def is_balanced(loads: Sequence[int], lam: float) -> bool:
    return imbalance_ratio(loads) < lam


def capacity(total: int, world: int, alpha: float) -> int:
    """m_α = α × (1/P) × Σ l  (Alg. 2), floored once (R1)."""
    return int(math.floor((alpha * float(total)) / float(world)))


def weight_transfer_plan(chunks: List[List[Chunk]], M: int) -> List[Tuple[int, int, int]]:
    """𝒲: W_i moves native(i) -> q for every device q != native(i) holding a chunk of i."""
    out = set()
    for e, A in enumerate(chunks):
        ng = native_device(e, M)
        for (d, _s, _t) in A:
            if d != ng:
                out.add((e, ng, d))
    return sorted(out)


def ep_plan(loads: Sequence[int], world: int, alpha: float = 1.0, fallback: bool = True) -> Plan:
    """Standard EP (Alg. 1): every expert's whole load on its native device."""
    loads = [int(x) for x in loads]
    N = len(loads)
    M = N // world
    chunks = [[(native_device(e, M), 0, le)] if le > 0 else [] for e, le in enumerate(loads)]
    ga = [0] * world
    for e, le in enumerate(loads):
        ga[native_device(e, M)] += le
    S = sum(loads)
    return Plan(N, world, chunks, ga, capacity(S, world, alpha), S, fallback, 0, [])


def _llas(ng: int, r: int, to: int, A: List[Chunk], ga: List[int], gp: List[int],
          cap: int, m: int, world: int) -> int:
    """Alg. 3.  Returns the number of force-assigns performed."""
    forces = 0
    while r > 0:
        o = sorted((g for g in range(world) if g != ng),             # P:492 (R5)
                   key=lambda g: (ga[g] + gp[g], g))
        if not o:
            raise PlannerError("spill with world size 1")
        assigned = False
        for cand in o:
            c = min(r, cap - ga[cand] - gp[cand])
            if c <= 0:                                               # R3
                continue
            if c < m and r > c:                                      # P:495-497 (R4)
                continue
            A.append((cand, to, to + c))
            ga[cand] += c
            r -= c
            to += c
            assigned = True
            break
        if not assigned:                                             # P:504-510 (R7)
            cand = o[0]
            A.append((cand, to, to + r))
            ga[cand] += r
            r = 0
            forces += 1
    return forces


def lla(loads: Sequence[int], world: int, alpha: float, min_chunk: int) -> Plan:
    """Alg. 2 with LLAS; no λ test."""
    loads = [int(x) for x in loads]
    N = len(loads)
    P = world
    M = N // P
    order = sorted(range(N), key=lambda e: (-loads[e], e))           # P:388 (R5)
    gn = [0] * P
    for e, le in enumerate(loads):
        gn[native_device(e, M)] += le
    gp = list(gn)
    ga = [0] * P
    S = sum(loads)
    cap = capacity(S, P, alpha)                                      # P:394 (R1)
    chunks: List[List[Chunk]] = [[] for _ in range(N)]
    forces = 0
    for i in order:
        e = loads[i]
        if e == 0:                                                   # R6
            continue
        ng = native_device(i, M)
        gp[ng] -= e
        na = cap - ga[ng] - gp[ng]
        A: List[Chunk] = []
        if na >= e:                                                  # P:402 Case 1
            A.append((ng, 0, e))
            ga[ng] += e
        elif na > 0:                                                 # P:406 Case 2 (R2)
            nc = min(na, e)
            to = nc
            A.append((ng, 0, nc))
            ga[ng] += nc
            r = e - nc
            forces += _llas(ng, r, to, A, ga, gp, cap, min_chunk, P)
        else:                                                        # P:414 Case 3
            forces += _llas(ng, e, 0, A, ga, gp, cap, min_chunk, P)
        chunks[i] = A
    return Plan(N, P, chunks, ga, cap, S, False, forces,
                weight_transfer_plan(chunks, M))


def plan(loads: Sequence[int], world: int, alpha: float = 1.0, min_chunk: int = 1024,
         lam: float = 1.3) -> Plan:
    """Alg. 4 planning steps: λ test, then LLA."""
    validate(loads, world, alpha, min_chunk, lam)
    S = sum(int(x) for x in loads)
    if S == 0 or is_balanced(loads, lam):                            # P:538-541 (R9)
        return ep_plan(loads, world, alpha, fallback=True)
    return lla(loads, world, alpha, min_chunk)


def max_device_load(p: Plan) -> int:
    return max(p.assigned) if p.assigned else 0
