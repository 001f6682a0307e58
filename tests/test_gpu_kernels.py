"""GPU kernel tests through the C ABI: device planner (bit-exact) and the tcgen05 grouped GEMMs."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_17111_b200 import llep
    return llep


def _same_plan(p, q):
    assert [list(A) for A in p.chunks] == [list(A) for A in q.chunks]
    assert p.assigned == q.assigned and p.capacity == q.capacity and p.total == q.total
    assert p.fallback == q.fallback and p.force_count == q.force_count
    assert p.transfers == q.transfers


def _plans_on_device(L, cases, ep=False):
    """Run llep_plan_device on every (C [P, N] int32, alpha, m, lam) case: one device buffer holds all
    load matrices and all output blobs, the launches are issued back to back on one stream (ctypes, no
    per-case synchronisation), and the blobs come back in one copy.  -> list of blob bytes."""
    import ctypes
    dev = torch.device("cuda:0")
    offs_in, offs_out, pos_in, pos_out = [], [], 0, 0
    for (C, _a, _m, _l) in cases:
        offs_in.append(pos_in)
        pos_in += C.size * 4
        offs_out.append(pos_out)
        pos_out += (L.plan_bytes(C.shape[1], C.shape[0]) + 15) // 16 * 16
    buf_in = np.zeros(max(pos_in, 4), dtype=np.uint8)
    for (C, *_), o in zip(cases, offs_in):
        buf_in[o:o + C.size * 4] = np.ascontiguousarray(C, dtype=np.int32).view(np.uint8).reshape(-1)
    d_in = torch.from_numpy(buf_in).to(dev)
    d_out = torch.zeros(max(pos_out, 16), dtype=torch.uint8, device=dev)
    s = L._stream_ptr()
    base_in, base_out = d_in.data_ptr(), d_out.data_ptr()
    f = L._lib.llep_plan_device
    for (C, a, m, lam), oi, oo in zip(cases, offs_in, offs_out):
        prm = L.params(a, m, lam)
        rc = f(base_in + oi, C.shape[1], C.shape[0], ctypes.byref(prm), int(ep), base_out + oo, s)
        assert rc == 0, L._lib.llep_last_error()
    out = d_out.cpu().numpy()
    return [out[o:o + L.plan_bytes(C.shape[1], C.shape[0])].tobytes() for (C, *_), o in zip(cases, offs_out)]


def test_device_planner_bit_exact(L):
    """10^4 random load matrices: device plan blob == host plan blob byte for byte, and == the oracle
    (O1) field by field (chunks in order, g_a, cap, S, fallback, force_count, 𝒲), for LLEP and EP."""
    from oracle import planner as O1
    rng = random.Random(77)
    cases = []
    while len(cases) < 10000:
        P = rng.choice([1, 2, 3, 4, 8, 8, 16, 32])
        M = rng.choice([1, 2, 4, 8, 16] + ([32, 64] if rng.random() < 0.05 else []))
        N = P * M
        if N > 1024:
            continue
        alpha = rng.choice([1.0, 1.0, 1.5, 2.0, rng.uniform(1, 3)])
        m = rng.choice([0, 1, 8, 64, 1024])
        lam = rng.choice([1.0, 1.3, 2.0])
        C = np.zeros((P, N), dtype=np.int32)
        for p in range(P):
            C[p] = [rng.randint(0, 30) for _ in range(N)]
            if rng.random() < 0.7:
                C[p, rng.randrange(N)] += rng.randint(100, 20000)
        cases.append((C, alpha, m, lam))
    for ep in (False, True):
        blobs = _plans_on_device(L, cases, ep=ep)
        for i, ((C, alpha, m, lam), blob) in enumerate(zip(cases, blobs)):
            l = C.sum(0).astype(np.int64)
            P = C.shape[0]
            dp = L.parse_plan(blob)
            hp = L.plan_host(l, P, alpha, m, lam, ep=ep)
            assert dp.raw == hp.raw, (i, P, C.shape[1], alpha, m, lam, ep)
            ref = O1.ep_plan(l, P, alpha, fallback=False) if ep else O1.plan(l.tolist(), P, alpha, m, lam)
            _same_plan(dp, ref)


def test_device_planner_bruteforce_box(L):
    """The brute-force box of SURVEY §8(c): every l in {0..7}^N for N <= 4 and P | N, α ∈ {1, 1.5, 2},
    m ∈ {0, 1, 2, 3, 8}, λ ∈ {1, 1.3, ∞} (≈ 6·10^5 plans): the device planner equals O1 on every field."""
    import itertools
    from oracle import planner as O1
    cases = []
    for N in (1, 2, 3, 4):
        for P in [p for p in (1, 2, 3, 4) if N % p == 0]:
            for l in itertools.product(range(8), repeat=N):
                C = np.zeros((P, N), dtype=np.int32)
                C[0] = l
                if P > 1:   # split the loads over the ranks (only column sums matter to the plan)
                    C[P - 1] = np.array(l) // 2
                    C[0] -= C[P - 1]
                for alpha in (1.0, 1.5, 2.0):
                    for m in (0, 1, 2, 3, 8):
                        for lam in (1.0, 1.3, float("inf")):
                            cases.append((C, alpha, m, lam))
    assert len(cases) > 500000
    for i0 in range(0, len(cases), 100000):
        part = cases[i0:i0 + 100000]
        blobs = _plans_on_device(L, part)
        for (C, alpha, m, lam), blob in zip(part, blobs):
            ref = O1.plan(C.sum(0).tolist(), C.shape[0], alpha, m, lam)
            _same_plan(L.parse_plan(blob), ref)


def _ref_gemm(mode, a, w, groups, nout, gate):
    out = torch.zeros((a.shape[0], nout), dtype=torch.float32, device=a.device)
    for (e, rb, n) in groups:
        x = a[rb:rb + n].float()
        if mode == 0:
            g = x @ w[e, :nout].float().T
            u = x @ w[e, nout:].float().T
            out[rb:rb + n] = torch.nn.functional.silu(g) * u
        else:
            out[rb:rb + n] = gate[rb:rb + n, None] * (x @ w[e].float().T)
    return out


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("mode,kdim,nout", [
    (0, 256, 512),    # TINY GEMM1 (BN=256)
    (1, 512, 256),    # TINY GEMM2
    (0, 2880, 2880),  # gpt-oss GEMM1 (BN=240: 120 gate + 120 up)
    (1, 2880, 2880),  # gpt-oss GEMM2 (BN=240)
    (0, 2048, 768),   # Qwen3 GEMM1
    (1, 768, 2048),   # Qwen3 GEMM2
    (0, 192, 200),    # ragged: masked tail tile, partial K block
    (1, 200, 136),
    (0, 128, 144),    # masked tail tiles at other widths
    (1, 256, 288),
    (0, 136, 264),
    (0, 7168, 2048),  # DeepSeek-V3 / Kimi-K2 GEMM1 (row f3: D=7168 -> 56 K-stages of 128)
    (1, 2048, 7168),  # DeepSeek-V3 / Kimi-K2 GEMM2 (nout 7168 = 28 tiles of 256)
    (0, 2048, 2048),  # F-head GEMM1
])
def test_grouped_gemm(L, mode, kdim, nout, pair):
    g = torch.Generator(device="cuda").manual_seed(kdim * 7 + nout)
    E = 3
    sizes = [1, 300, 0, 129, 128, 77, 600, 256, 385]
    ra = 256 if pair else 128  # 2-CTA pair tiles are 256 rows: group bases 256-aligned
    groups, rb = [], 0
    for i, n in enumerate(sizes):
        if n == 0:
            continue
        groups.append((i % E, rb, n))
        rb += (n + ra - 1) // ra * ra
    rows = rb + 128
    a = (torch.randn((rows, kdim), generator=g, device="cuda") ).to(torch.bfloat16)
    wr = 2 * nout if mode == 0 else nout
    w = (torch.randn((E, wr, kdim), generator=g, device="cuda") / kdim ** 0.5).to(torch.bfloat16)
    gate = torch.rand((rows,), generator=g, device="cuda") if mode == 1 else None
    out = L.grouped_gemm(mode, a, w, groups, nout, gate, pair=pair)
    torch.cuda.synchronize()
    ref = _ref_gemm(mode, a, w, groups, nout, gate)
    for (e, rb, n) in groups:
        y, r = out[rb:rb + n].float(), ref[rb:rb + n]
        err = (y - r).abs().max().item() / max(r.abs().max().item(), 1e-6)
        l2 = ((y - r).norm() / r.norm().clamp_min(1e-12)).item()
        assert err < 2e-2 and l2 < 5e-3, (e, rb, n, err, l2)
    # rows outside groups are untouched (zeros)
    mask = torch.ones(rows, dtype=torch.bool, device="cuda")
    for (e, rb, n) in groups:
        mask[rb:rb + n] = False
    assert out[mask].abs().max().item() == 0.0


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("kind,kdim,nout", [
    (0, 2880, 2880),   # dA = dY · W_down   (W_down [D][H])
    (0, 5760, 2880),   # dX = dGU · W13     (W13 [2H][D])
    (0, 256, 512),
    (1, 2880, 2880),   # dW_down = dYᵀ · a  (mdim = D, nout = H)
    (1, 5760, 2880),   # dW13 = dGUᵀ · X    (mdim = 2H, nout = D)
    (1, 512, 256),
])
def test_gemm_bwd(L, kind, kdim, nout, pair):
    """Backward GEMMs with MN-major UMMA operands vs a plain fp32 torch reference."""
    g = torch.Generator(device="cuda").manual_seed(kind * 100 + kdim + nout)
    E = 3
    sizes = [1, 300, 129, 600, 256, 64, 65, 128] + ([9000] if kind == 1 else [])   # 9000 rows: split-K path
    groups, rb = [], 0
    for i, n in enumerate(sizes):
        groups.append((i % E, rb, n))
        rb += (n + 255) // 256 * 256
    rows = rb
    if kind == 0:
        a = torch.randn((rows, kdim), generator=g, device="cuda").to(torch.bfloat16)
        w = (torch.randn((E, kdim, nout), generator=g, device="cuda") / kdim ** 0.5).to(torch.bfloat16)
        out = L.gemm_bwd(0, a, w, groups, nout, kdim, E, pair=pair)
        torch.cuda.synchronize()
        for (e, rb, n) in groups:
            ref = a[rb:rb + n].float() @ w[e].float()
            y = out[rb:rb + n].float()
            err = ((y - ref).norm() / ref.norm()).item()
            assert err < 5e-3 and (y - ref).abs().max().item() / ref.abs().max().item() < 2e-2, (e, n, err)
    else:
        mdim = kdim
        a = torch.randn((rows, mdim), generator=g, device="cuda").to(torch.bfloat16)
        b = torch.randn((rows, nout), generator=g, device="cuda").to(torch.bfloat16)
        for (e, rb, n) in groups:  # zero the padding rows of each group
            a[rb + n:rb + (n + 255) // 256 * 256] = 0
            b[rb + n:rb + (n + 255) // 256 * 256] = 0
        gl = [(i, rb, n) for i, (e, rb, n) in enumerate(groups)]
        out = L.gemm_bwd(1, a, b, gl, nout, mdim, len(gl), pair=pair)
        torch.cuda.synchronize()
        for (i, rb, n) in gl:
            ref = a[rb:rb + n].float().T @ b[rb:rb + n].float()
            y = out[i]
            err = ((y - ref).norm() / ref.norm()).item()
            assert err < 1e-4, (i, n, err)
