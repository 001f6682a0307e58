"""Thin ctypes binding of the C-ABI library `libllep.so` (include/llep.h).

Argument marshalling only: every step of the layer runs in the library's CUDA kernels.  torch is
used for device memory, streams and (for P > 1) the process group that carries the 64-byte IPC
handles of the symmetric arenas.  There is no CPU fallback: if the library is missing, importing
this module raises.
"""
from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LLEP_LIB") or os.path.join(_PKG, "libllep.so")  # LLEP_LIB: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2601_17111_b200.build`")
_lib = ctypes.CDLL(LIB_PATH)

STATUS = {0: "OK", 1: "INVALID", 2: "PLAN", 3: "ROUTING", 4: "NOMEM", 5: "CUDA", 6: "COMM"}


class LLEPError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"LLEP_ERR_{STATUS.get(code, code)}: {msg}")
        self.code = code


class Params(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("min_chunk", ctypes.c_int64), ("lambda_", ctypes.c_double)]


class Shape(ctypes.Structure):
    _fields_ = [("n_experts", ctypes.c_int32), ("top_k", ctypes.c_int32), ("d_model", ctypes.c_int32),
                ("d_ff", ctypes.c_int32), ("world_size", ctypes.c_int32)]


PHASES = ("route", "exchange", "plan", "dispatch", "gemm1", "gemm2", "combine")


class Stats(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 7), ("calls", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("gemm_rows", ctypes.c_int64)]


class Requirements(ctypes.Structure):
    _fields_ = [("rows_needed", ctypes.c_int64), ("foreign_needed", ctypes.c_int32), ("fits", ctypes.c_int32),
                ("my_rows", ctypes.c_int64), ("my_groups", ctypes.c_int32), ("fallback_ep", ctypes.c_int32),
                ("force_count", ctypes.c_int32), ("n_transfers", ctypes.c_int32),
                ("grad_slots_needed", ctypes.c_int32)]


_vp, _i32, _i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_SIGS = {
    "llep_last_error": (ctypes.c_char_p, []),
    "llep_version": (ctypes.c_char_p, []),
    "llep_plan_bytes": (ctypes.c_size_t, [_i32, _i32]),
    "llep_plan": (ctypes.c_int, [_vp, _i32, _i32, ctypes.POINTER(Params), _vp]),
    "llep_plan_ep": (ctypes.c_int, [_vp, _i32, _i32, ctypes.POINTER(Params), _vp]),
    "llep_plan_device": (ctypes.c_int, [_vp, _i32, _i32, ctypes.POINTER(Params), _i32, _vp, _vp]),
    "llep_context_create": (ctypes.c_int, [ctypes.POINTER(Shape), _i32, _i32, _i64, ctypes.POINTER(_vp)]),
    "llep_context_destroy": (None, [_vp]),
    "llep_context_ipc_handle": (ctypes.c_int, [_vp, _vp]),
    "llep_context_open_peers": (ctypes.c_int, [_vp, _vp, _i32]),
    "llep_context_reserve": (ctypes.c_int, [_vp, _i64, _i32, _i32]),
    "llep_context_enable_backward": (ctypes.c_int, [_vp]),
    "llep_moe_backward": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "llep_context_device_bytes": (_i64, [_vp]),
    "llep_context_set_memory_cap": (ctypes.c_int, [_vp, _i64]),
    "llep_context_set_token_order": (ctypes.c_int, [_vp, _i32]),
    "llep_prepare": (ctypes.c_int, [_vp, _vp, _i64, ctypes.POINTER(Params), _i32, _vp,
                                    ctypes.POINTER(Requirements), _vp]),
    "llep_moe_forward": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "llep_moe_layer": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp, ctypes.POINTER(Params), _i32, _vp, _vp,
                                      _vp]),
    "llep_moe_forward_train": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp]),
    "llep_moe_backward_saved": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp,
                                               _vp, _vp, _vp]),
    "llep_debug_copy": (ctypes.c_int, [_vp, _i32, _vp, _i64, _vp]),
    "llep_context_set_timing": (ctypes.c_int, [_vp, _i32]),
    "llep_context_check": (ctypes.c_int, [_vp, _vp]),
    "llep_context_stats": (ctypes.c_int, [_vp, ctypes.c_void_p, _i32]),
    "llep_gemm_bwd": (ctypes.c_int, [_i32, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _i32, _vp, _vp]),
    "llep_grouped_gemm": (ctypes.c_int, [_i32, _vp, _i64, _i32, _vp, _i32, _i32, _vp, _i32, _vp, _vp, _vp]),
    "llep_router": (ctypes.c_int, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
}
EXPORTS = tuple(_SIGS)
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

ORDER_RANK_MAJOR, ORDER_CHUNK_ALIGNED = 0, 1
DBG_LOAD_MATRIX, DBG_SLOT_DST, DBG_GROUPS, DBG_RECV_X, DBG_ACT, DBG_Y, DBG_LOCAL_RANK, DBG_RECV_G = range(1, 9)


def _check(code: int) -> None:
    if code != 0:
        raise LLEPError(code, _lib.llep_last_error().decode())


def version() -> str:
    return _lib.llep_version().decode()


def params(alpha: float = 1.0, min_chunk: int = 1024, lam: float = 1.3) -> Params:
    return Params(float(alpha), int(min_chunk), float(lam))


# ------------------------------------------------------------------------------ plans
HEADER = struct.Struct("<iiiiii q q q iiii")


@dataclass
class Plan:
    n_experts: int
    world: int
    fallback: bool
    force_count: int
    n_transfers: int
    total: int
    capacity: int
    max_assigned: int
    assigned: List[int]
    chunks: List[List[Tuple[int, int, int]]]
    transfers: List[Tuple[int, int, int]]
    raw: bytes


def plan_bytes(n_experts: int, world: int) -> int:
    return int(_lib.llep_plan_bytes(n_experts, world))


def parse_plan(blob: bytes) -> Plan:
    (N, P, MC, fb, forces, ntr, S, cap, mx, oa, on, oc, orr) = HEADER.unpack_from(blob, 0)
    assigned = list(np.frombuffer(blob, dtype=np.int64, count=P, offset=oa))
    nch = np.frombuffer(blob, dtype=np.int32, count=N, offset=on)
    ch = np.frombuffer(blob, dtype=np.int32, count=N * MC * 3, offset=oc).reshape(N, MC, 3)
    rep = np.frombuffer(blob, dtype=np.uint8, count=N * P, offset=orr).reshape(N, P)
    chunks = [[tuple(int(v) for v in ch[e, c]) for c in range(int(nch[e]))] for e in range(N)]
    M = N // P
    transfers = [(e, e // M, d) for e in range(N) for d in range(P) if rep[e, d]]
    return Plan(N, P, bool(fb), forces, ntr, S, cap, mx, [int(a) for a in assigned], chunks, transfers,
                bytes(blob))


def plan_host(loads: Sequence[int], world: int, alpha: float = 1.0, min_chunk: int = 1024,
              lam: float = 1.3, ep: bool = False) -> Plan:
    """llep_plan / llep_plan_ep on the host."""
    l = np.ascontiguousarray(np.asarray(loads, dtype=np.int64))
    N = int(l.size)
    nb = plan_bytes(N, world)
    if nb == 0:
        raise LLEPError(1, "N and P must be >= 1")
    buf = (ctypes.c_uint8 * nb)()
    f = _lib.llep_plan_ep if ep else _lib.llep_plan
    _check(f(l.ctypes.data, N, world, ctypes.byref(params(alpha, min_chunk, lam)), buf))
    return parse_plan(bytes(buf))


def _stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def plan_device(load_matrix, world: int, alpha: float = 1.0, min_chunk: int = 1024, lam: float = 1.3,
                ep: bool = False, out=None):
    """llep_plan_device on a [P, N] int32 CUDA tensor -> uint8 CUDA tensor (the plan blob)."""
    import torch
    P, N = load_matrix.shape
    assert P == world and load_matrix.dtype == torch.int32 and load_matrix.is_cuda
    lm = load_matrix.contiguous()
    if out is None:
        out = torch.empty(plan_bytes(N, P), dtype=torch.uint8, device=lm.device)
    _check(_lib.llep_plan_device(lm.data_ptr(), N, P, ctypes.byref(params(alpha, min_chunk, lam)),
                                 int(ep), out.data_ptr(), _stream_ptr()))
    return out


# ------------------------------------------------------------------------------ context
def _max_over_group(v: int, group) -> int:
    import torch.distributed as dist
    allv: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(allv, v, group=group)
    return max(allv)


class Context:
    """One rank's LLEP context: scratch, symmetric arena, peer mappings."""

    def __init__(self, n_experts: int, top_k: int, d_model: int, d_ff: int, world: int, rank: int,
                 device: int, max_tokens: int, group=None):
        import torch
        self.shape = Shape(n_experts, top_k, d_model, d_ff, world)
        self.N, self.K, self.D, self.H, self.P, self.rank = n_experts, top_k, d_model, d_ff, world, rank
        self.M = n_experts // world
        self.device = device
        self.group = group
        if world > 1:   # the arenas must be symmetric: every rank sizes its context for the largest B
            max_tokens = _max_over_group(int(max_tokens), group)
        self.max_tokens = max_tokens
        h = _vp()
        torch.cuda.set_device(device)
        _check(_lib.llep_context_create(ctypes.byref(self.shape), rank, device, max_tokens, ctypes.byref(h)))
        self._h = h
        self.last_req: Optional[Requirements] = None
        if world > 1:
            self.exchange_handles()

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            _lib.llep_context_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- symmetric arena
    def exchange_handles(self) -> None:
        import torch.distributed as dist
        buf = (ctypes.c_uint8 * 64)()
        _check(_lib.llep_context_ipc_handle(self._h, buf))
        mine = bytes(buf)
        allh: list = [None] * self.P
        dist.all_gather_object(allh, mine, group=self.group)
        blob = b"".join(allh)
        _check(_lib.llep_context_open_peers(self._h, blob, self.P))

    def reserve(self, rows: int, foreign: int, grad_slots: int = 0) -> None:
        _check(_lib.llep_context_reserve(self._h, int(rows), int(foreign), int(grad_slots)))
        if self.P > 1:
            self.exchange_handles()

    def enable_backward(self) -> None:
        """Row f1: arena regions for dout rows and returned weight-gradient partials (collective)."""
        _check(_lib.llep_context_enable_backward(self._h))
        if self.P > 1:
            self.exchange_handles()

    def check(self) -> None:
        """llep_context_check: synchronise and raise the sticky device-side error, if any."""
        _check(_lib.llep_context_check(self._h, _stream_ptr()))

    def set_timing(self, on: bool = True) -> None:
        _check(_lib.llep_context_set_timing(self._h, int(on)))

    def stats(self, reset: bool = False) -> dict:
        st = Stats()
        _check(_lib.llep_context_stats(self._h, ctypes.byref(st), int(reset)))
        return {"ms": dict(zip(PHASES, list(st.ms))), "calls": int(st.calls),
                "kernel_launches": int(st.kernel_launches), "gemm_rows": int(st.gemm_rows)}

    def set_token_order(self, order: str) -> None:
        """"chunk_aligned" (default, reading R11') or "rank_major" (R11): the global token order the
        plan's chunk ranges index.  Same on every rank; outputs identical, link bytes differ."""
        code = {"rank_major": ORDER_RANK_MAJOR, "chunk_aligned": ORDER_CHUNK_ALIGNED}[order]
        if self.P > 1:   # collective: every rank must address peers' rows with the same order
            import torch.distributed as dist
            allo: list = [None] * self.P
            dist.all_gather_object(allo, code, group=self.group)
            if len(set(allo)) != 1:
                raise LLEPError(1, f"llep_context_set_token_order: ranks disagree on the token order ({allo})")
        _check(_lib.llep_context_set_token_order(self._h, code))

    def set_memory_cap(self, nbytes: int) -> None:
        _check(_lib.llep_context_set_memory_cap(self._h, int(nbytes)))

    def device_bytes(self) -> int:
        return int(_lib.llep_context_device_bytes(self._h))

    # -- the hot path
    def prepare(self, topk_ids, alpha=1.0, min_chunk=1024, lam=1.3, ep=False, plan_out=None):
        import torch
        assert topk_ids.dtype == torch.int32 and topk_ids.is_cuda and topk_ids.is_contiguous()
        if plan_out is None:
            plan_out = torch.empty(plan_bytes(self.N, self.P), dtype=torch.uint8, device=topk_ids.device)
        req = Requirements()
        _check(_lib.llep_prepare(self._h, topk_ids.data_ptr(), topk_ids.shape[0],
                                 ctypes.byref(params(alpha, min_chunk, lam)), int(ep), plan_out.data_ptr(),
                                 ctypes.byref(req), _stream_ptr()))
        if not req.fits:
            # identical on every rank (replicated plan): grow symmetrically, re-map peers
            self.reserve(int(req.rows_needed), int(req.foreign_needed), int(req.grad_slots_needed))
            req.fits = 1
        self.last_req = req
        return plan_out, req

    def forward(self, x, topk_ids, topk_w, w13, w2, plan, out=None):
        import torch
        B = x.shape[0]
        for t, dt in ((x, torch.bfloat16), (topk_ids, torch.int32), (topk_w, torch.float32),
                      (w13, torch.bfloat16), (w2, torch.bfloat16)):
            assert t.dtype == dt and t.is_cuda and t.is_contiguous(), (t.dtype, dt)
        assert w13.shape == (self.M, 2 * self.H, self.D) and w2.shape == (self.M, self.D, self.H)
        if out is None:
            out = torch.empty((B, self.D), dtype=torch.bfloat16, device=x.device)
        _check(_lib.llep_moe_forward(self._h, x.data_ptr(), topk_ids.data_ptr(), topk_w.data_ptr(), B,
                                     w13.data_ptr(), w2.data_ptr(), plan.data_ptr(), out.data_ptr(),
                                     _stream_ptr()))
        return out

    def forward_train(self, x, topk_ids, topk_w, w13, w2, plan, out=None, gu=None):
        """llep_moe_forward_train: forward + this rank's raw [g | u] pre-activations saved for
        backward(..., gu=...).  Returns (out, gu); gu [rows_needed, 2H] bf16 unless given."""
        import torch
        B = x.shape[0]
        for t, dt in ((x, torch.bfloat16), (topk_ids, torch.int32), (topk_w, torch.float32),
                      (w13, torch.bfloat16), (w2, torch.bfloat16)):
            assert t.dtype == dt and t.is_cuda and t.is_contiguous(), (t.dtype, dt)
        assert w13.shape == (self.M, 2 * self.H, self.D) and w2.shape == (self.M, self.D, self.H)
        if out is None:
            out = torch.empty((B, self.D), dtype=torch.bfloat16, device=x.device)
        if gu is None:
            rows = int(self.last_req.rows_needed) if self.last_req is not None else 0
            gu = torch.empty((max(rows, 1), 2 * self.H), dtype=torch.bfloat16, device=x.device)
        assert gu.dtype == torch.bfloat16 and gu.is_contiguous() and gu.shape[1] == 2 * self.H
        _check(_lib.llep_moe_forward_train(self._h, x.data_ptr(), topk_ids.data_ptr(), topk_w.data_ptr(), B,
                                           w13.data_ptr(), w2.data_ptr(), plan.data_ptr(), out.data_ptr(),
                                           gu.data_ptr(), gu.shape[0], _stream_ptr()))
        return out, gu

    def backward(self, x, topk_ids, topk_w, dout, w13, w2, plan, dx=None, dgates=None, dw13=None, dw2=None,
                 gu=None):
        """llep_moe_backward under `plan` (from prepare on these topk_ids): returns
        (dx [B, D] bf16, dgates [B, K] fp32, dw13 [M, 2H, D] fp32, dw2 [M, D, H] fp32)."""
        import torch
        B = x.shape[0]
        dev = x.device
        assert dout.dtype == torch.bfloat16 and dout.is_contiguous() and dout.shape == x.shape
        dx = torch.empty_like(x) if dx is None else dx
        dgates = torch.empty((B, self.K), dtype=torch.float32, device=dev) if dgates is None else dgates
        dw13 = torch.empty((self.M, 2 * self.H, self.D), dtype=torch.float32, device=dev) if dw13 is None else dw13
        dw2 = torch.empty((self.M, self.D, self.H), dtype=torch.float32, device=dev) if dw2 is None else dw2
        if gu is not None:   # pre-activations saved by forward_train under the same plan
            assert gu.dtype == torch.bfloat16 and gu.is_contiguous() and gu.shape[1] == 2 * self.H
            _check(_lib.llep_moe_backward_saved(self._h, x.data_ptr(), topk_ids.data_ptr(), topk_w.data_ptr(),
                                                dout.data_ptr(), B, w13.data_ptr(), w2.data_ptr(), plan.data_ptr(),
                                                gu.data_ptr(), gu.shape[0], dx.data_ptr(), dgates.data_ptr(),
                                                dw13.data_ptr(), dw2.data_ptr(), _stream_ptr()))
            return dx, dgates, dw13, dw2
        _check(_lib.llep_moe_backward(self._h, x.data_ptr(), topk_ids.data_ptr(), topk_w.data_ptr(),
                                      dout.data_ptr(), B, w13.data_ptr(), w2.data_ptr(), plan.data_ptr(),
                                      dx.data_ptr(), dgates.data_ptr(), dw13.data_ptr(), dw2.data_ptr(),
                                      _stream_ptr()))
        return dx, dgates, dw13, dw2

    def layer(self, x, topk_ids, topk_w, w13, w2, alpha=1.0, min_chunk=1024, lam=1.3, ep=False,
              plan_out=None, out=None):
        """llep_moe_layer: prepare + forward in one call with no host synchronisation (CUDA-graph
        capturable; the plan is recomputed on the device each replay).  The arena must already hold the
        plan (reserve() first); an overflow surfaces at the next check()."""
        import torch
        B = x.shape[0]
        for t, dt in ((x, torch.bfloat16), (topk_ids, torch.int32), (topk_w, torch.float32),
                      (w13, torch.bfloat16), (w2, torch.bfloat16)):
            assert t.dtype == dt and t.is_cuda and t.is_contiguous(), (t.dtype, dt)
        assert w13.shape == (self.M, 2 * self.H, self.D) and w2.shape == (self.M, self.D, self.H)
        if plan_out is None:
            plan_out = torch.empty(plan_bytes(self.N, self.P), dtype=torch.uint8, device=x.device)
        if out is None:
            out = torch.empty((B, self.D), dtype=torch.bfloat16, device=x.device)
        self._params = params(alpha, min_chunk, lam)   # kept alive with the context (graph replays)
        _check(_lib.llep_moe_layer(self._h, x.data_ptr(), topk_ids.data_ptr(), topk_w.data_ptr(), B,
                                   w13.data_ptr(), w2.data_ptr(), ctypes.byref(self._params), int(ep),
                                   plan_out.data_ptr(), out.data_ptr(), _stream_ptr()))
        return out

    def __call__(self, x, topk_ids, topk_w, w13, w2, alpha=1.0, min_chunk=1024, lam=1.3, ep=False,
                 plan_out=None, out=None):
        """One MoE-layer forward (Alg. 4): prepare (histogram, exchange, plan, layout) + forward."""
        plan, _ = self.prepare(topk_ids, alpha, min_chunk, lam, ep, plan_out)
        return self.forward(x, topk_ids, topk_w, w13, w2, plan, out)

    def debug(self, what: int, n: int, dtype):
        import torch
        t = torch.empty(n, dtype=dtype, device=f"cuda:{self.device}")
        _check(_lib.llep_debug_copy(self._h, what, t.data_ptr(), n, _stream_ptr()))
        return t


def router(x, w_router, top_k: int, logits: bool = False, out=None):
    """llep_router (row f4, Eq. 2): x [B, D] bf16, w_router [N, D] bf16 (= W_rᵀ) on the current
    device -> (topk_ids int32 [B, K], topk_w fp32 [B, K]) [+ logits fp32 [B, N] if logits=True].
    `out` = (ids, gates) preallocated tensors, optional."""
    import torch
    B, D = x.shape
    N = w_router.shape[0]
    if out is None:
        ids = torch.empty((B, top_k), dtype=torch.int32, device=x.device)
        gates = torch.empty((B, top_k), dtype=torch.float32, device=x.device)
    else:
        ids, gates = out
    z = torch.empty((B, N), dtype=torch.float32, device=x.device) if logits else None
    _check(_lib.llep_router(x.data_ptr(), w_router.data_ptr(), B, D, N, top_k, ids.data_ptr(), gates.data_ptr(),
                            z.data_ptr() if z is not None else None, _stream_ptr()))
    return (ids, gates, z) if logits else (ids, gates)


def grouped_gemm(mode: int, a, w, groups: Sequence[Tuple[int, int, int]], nout: int, gate=None, out=None,
                 pair: bool = False):
    """llep_grouped_gemm: groups = [(expert, row_base, n_rows)] (host), a [rows, kdim] bf16,
    mode 0: w [E, 2*nout, kdim] -> SwiGLU [rows, nout]; mode 1: w [E, nout, kdim] -> gate*(a wᵀ).
    pair=True: 2-CTA (cta_group::2) 256-row tiles, row bases must be multiples of 256."""
    import torch
    rows, kdim = a.shape
    if out is None:
        out = torch.zeros((rows, nout), dtype=torch.bfloat16, device=a.device)
    g = np.asarray([[e, rb, n, 0] for (e, rb, n) in groups], dtype=np.int32).reshape(-1)
    g = np.ascontiguousarray(g)
    _check(_lib.llep_grouped_gemm(mode | (2 if pair else 0), a.data_ptr(), rows, kdim, w.data_ptr(), w.shape[0], nout,
                                  g.ctypes.data, len(groups), gate.data_ptr() if gate is not None else None,
                                  out.data_ptr(), _stream_ptr()))
    return out


def gemm_bwd(kind: int, a, b, groups: Sequence[Tuple[int, int, int]], nout: int, kdim_or_mdim: int,
             n_weights: int, out=None, pair: bool = False):
    """llep_gemm_bwd (see llep.h): kind 0 -> bf16 [rows, nout]; kind 1 -> fp32 [n_weights, mdim, nout]."""
    import torch
    rows = a.shape[0]
    if out is None:
        if kind == 0:
            out = torch.zeros((rows, nout), dtype=torch.bfloat16, device=a.device)
        else:
            out = torch.zeros((n_weights, kdim_or_mdim, nout), dtype=torch.float32, device=a.device)
    g = np.ascontiguousarray(np.asarray([[e, rb, n, 0] for (e, rb, n) in groups], dtype=np.int32).reshape(-1))
    _check(_lib.llep_gemm_bwd(kind | (2 if pair else 0), a.data_ptr(), b.data_ptr(), rows, kdim_or_mdim, nout, n_weights,
                              g.ctypes.data, len(groups), out.data_ptr(), _stream_ptr()))
    return out
