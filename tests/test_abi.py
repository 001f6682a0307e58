"""The C-ABI library loads, exports every symbol llep.h declares, and its HOST planner
(llep_plan / llep_plan_ep, no GPU needed) is bit-identical to the oracle -- CPU only."""
import ctypes
import os
import random
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2601_17111_b200 import build
    build.build()
    from paper_2601_17111_b200 import llep
    return llep


def test_exports_match_header(L):
    hdr = open(os.path.join(ROOT, "include", "llep.h")).read()
    declared = set(re.findall(r"^(?:const\s+)?[a-z_0-9]+\s*\*?\s*(llep_[a-z_0-9]+)\(", hdr, re.M))
    assert declared, "no declarations parsed"
    import ctypes
    lib = ctypes.CDLL(L.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(L.EXPORTS)


def test_plan_bytes_and_header(L):
    assert L.plan_bytes(128, 8) > 0 and L.plan_bytes(0, 8) == 0
    p = L.plan_host([10, 0, 0, 0], 2, 1.0, 1, 1.0)
    assert p.n_experts == 4 and p.world == 2 and p.chunks[0] == [(0, 0, 5), (1, 5, 10)]
    assert p.assigned == [5, 5] and p.transfers == [(0, 0, 1)] and p.capacity == 5


def test_host_plan_errors(L):
    for args in [([1, 2, 3], 2, 1.0, 0, 1.3), ([1, 2], 2, 0.5, 0, 1.3), ([1, 2], 2, 1.0, 0, 0.9),
                 ([1, -2], 2, 1.0, 0, 1.3), ([1, 2], 2, 1.0, -1, 1.3)]:
        with pytest.raises(L.LLEPError) as ei:
            L.plan_host(*args)
        assert ei.value.code == 1


def _same(p, q):
    assert [list(A) for A in p.chunks] == [list(A) for A in q.chunks]
    assert p.assigned == q.assigned and p.capacity == q.capacity and p.total == q.total
    assert p.fallback == q.fallback and p.force_count == q.force_count
    assert p.transfers == q.transfers


def test_host_plan_matches_oracle_fuzz(L):
    from oracle import planner as O1
    rng = random.Random(2024)
    for i in range(4000):
        P = rng.choice([1, 2, 3, 4, 8, 16])
        M = rng.choice([1, 2, 4, 8, 16])
        N = P * M
        alpha = rng.choice([1.0, 1.0, 1.5, 2.0, rng.uniform(1, 3)])
        m = rng.choice([0, 1, 2, 8, 64, 1024])
        lam = rng.choice([1.0, 1.3, 2.0])
        kind = rng.randrange(3)
        if kind == 0:
            l = [rng.randint(0, 60) for _ in range(N)]
        elif kind == 1:
            l = [rng.randint(0, 20) for _ in range(N)]
            for _ in range(rng.randint(1, 3)):
                l[rng.randrange(N)] += rng.randint(100, 20000)
        else:
            l = [rng.choice([0, 1, 5, 3000]) for _ in range(N)]
        _same(L.plan_host(l, P, alpha, m, lam), O1.plan(l, P, alpha, m, lam))
        _same(L.plan_host(l, P, alpha, m, lam, ep=True), O1.ep_plan(l, P, alpha, fallback=False))


def test_host_plan_golden_and_paper_configs(L, golden_dir):
    import json
    from oracle import planner as O1
    from synth import workload as W
    g = json.load(open(os.path.join(golden_dir, "planner_traces.json")))
    for c in g["cases"]:
        p = L.plan_host(c["loads"], c["world"], c["alpha"], c["min_chunk"], 1.0)
        assert [[list(x) for x in A] for A in p.chunks] == c["chunks"]
        assert p.force_count == c["force_count"]
    for name in ("tiny", "g20", "g120", "q3"):
        sh = W.CONFIGS[name]
        for pct, y in [(None, 0), (30, 1), (50, 4), (80, 16), (95, 1)]:
            if y > sh.n_experts:
                continue
            cnt = W.slot_counts(sh.n_experts, sh.tokens_per_rank * sh.top_k, pct, y)
            for P in (1, 2, 4, 8):
                if sh.n_experts % P:
                    continue
                l = (cnt * P).tolist()
                _same(L.plan_host(l, P), O1.plan(l, P))


def test_context_create_validation(L):
    """Shape rules of llep_context_create are checked before any CUDA call: CPU-testable."""
    import ctypes
    bad = [
        (6, 2, 256, 512, 4),     # N % P != 0
        (8, 9, 256, 512, 2),     # K > N
        (8, 0, 256, 512, 2),     # K < 1
        (8, 2, 250, 512, 2),     # D % 8 != 0
        (8, 2, 256, 4, 2),       # H < 8
        (64, 2, 256, 512, 64),   # P > 32
        (2048, 2, 256, 512, 2),  # N > 1024
    ]
    for (N, K, D, H, P) in bad:
        sh = L.Shape(N, K, D, H, P)
        h = ctypes.c_void_p()
        code = L._lib.llep_context_create(ctypes.byref(sh), 0, 0, 16, ctypes.byref(h))
        assert code == 1, (N, K, D, H, P, code)
        assert L._lib.llep_last_error()
    sh = L.Shape(8, 2, 256, 512, 2)
    h = ctypes.c_void_p()
    assert L._lib.llep_context_create(ctypes.byref(sh), 2, 0, 16, ctypes.byref(h)) == 1   # rank >= P


def test_plan_bytes_formula(L):
    """Blob layout: header, g_a [P] int64, n_chunks [N] int32, chunks [N][P+1] x 12 B, replica [N][P]."""
    for N, P in [(8, 2), (128, 8), (384, 32), (1, 1)]:
        a8 = lambda x: (x + 7) // 8 * 8
        off = a8(64)
        off = a8(off + 8 * P)
        off = a8(off + 4 * N)
        off = a8(off + 12 * N * (P + 1))
        off = a8(off + N * P)
        assert L.plan_bytes(N, P) == off


def test_router_validation(L):
    """llep_router rejects out-of-range arguments with LLEP_ERR_INVALID before touching the device;
    an empty batch is a no-op that returns OK (no CUDA call)."""
    lib = L._lib
    buf = (ctypes.c_uint16 * 64)()
    ids = (ctypes.c_int32 * 8)()
    g = (ctypes.c_float * 8)()
    p = ctypes.addressof(buf)
    cases = [
        (p, p, 4, 64, 0, 1),      # N < 1
        (p, p, 4, 64, 513, 2),    # N > 512
        (p, p, 4, 64, 8, 0),      # K < 1
        (p, p, 4, 64, 8, 9),      # K > N
        (p, p, 4, 64, 32, 17),    # K > 16
        (p, p, 4, 60, 8, 2),      # D % 8
        (p, p, -1, 64, 8, 2),     # negative batch
        (None, p, 4, 64, 8, 2),   # null x
    ]
    for (x, w, B, D, N, K) in cases:
        assert lib.llep_router(x, w, B, D, N, K, ctypes.addressof(ids), ctypes.addressof(g), None, None) == 1
        assert lib.llep_last_error()
    assert lib.llep_router(None, None, 0, 64, 8, 2, None, None, None, None) == 0


def test_missing_library_fails_loudly(tmp_path):
    """The binding has no CPU fallback: without the compiled library the import raises."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LLEP_LIB=str(tmp_path / "no_such_libllep.so"))
    r = subprocess.run([sys.executable, "-c", "from paper_2601_17111_b200 import llep"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and ("OSError" in r.stderr or "ImportError" in r.stderr or "not found" in r.stderr), r.stderr[-500:]
