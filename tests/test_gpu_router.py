"""Row f4: the router of Eq. 2 on the GPU (llep_router, router.cu) vs the float64
oracle O6.  Inputs are the seeded synth tokens and router weights (exact bf16 values).

Parity has two parts ("router"):
  * the logits z = x·W_r: each within an fp32-accumulation bound of the float64 value;
  * the decision (top-K ids, their order) and the gates, taken in the kernel's precision: O6 applied
    to the kernel's own fp32 logits must reproduce the kernel's ids exactly and its gates to fp32
    rounding.  Against the float64 logits the ids must agree wherever the float64 margin between the
    competing experts exceeds twice the logit bound (a smaller margin is a legitimate near tie).
"""
import numpy as np
import pytest

from synth import workload as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_17111_b200 import llep
    return llep


def _inputs(B, D, N, seed, scale=1.0):
    dev = torch.device("cuda:0")
    x = W.tokens_torch(B, D, 0, dev, seed)
    w = W.router_weight_torch(N, D, dev, scale=scale, seed=seed)
    return x, w


def _oracle_logits(B, D, N, seed, rows, scale=1.0):
    from oracle import router as O6
    x = W.bf16_bits_to_f64(W.token_rows_bits(rows, D, 0, seed))
    w = W.bf16_bits_to_f64(W.router_weight_bits(N, D, scale=scale, seed=seed))
    z = O6.logits(x, w.T)                     # W_r = wᵀ [D, N] (reading R33)
    bound = 1e-5 * (np.abs(x) @ np.abs(w.T)) + 1e-30   # fp32 accumulation of D exact products
    return z, bound


def _check(L, B, D, N, K, seed, sample=None, scale=1.0):
    from oracle import router as O6
    x, w = _inputs(B, D, N, seed, scale)
    ids, gates, z = L.router(x, w, K, logits=True)
    ids2, gates2 = L.router(x, w, K)
    torch.cuda.synchronize()
    assert torch.equal(ids, ids2) and torch.equal(gates, gates2), "logits copy must not change the result"
    ids, gates, z = ids.cpu().numpy(), gates.cpu().numpy(), z.cpu().numpy().astype(np.float64)
    rows = np.arange(B) if sample is None else np.unique(np.concatenate(
        [np.arange(min(B, 64)), np.arange(max(0, B - 64), B), np.random.default_rng(seed).choice(B, sample)]))
    # 1. logits within the fp32 bound of float64
    zo, bound = _oracle_logits(B, D, N, seed, rows, scale)
    assert np.all(np.abs(z[rows] - zo) <= bound), np.max(np.abs(z[rows] - zo) / bound)
    # 2. decision + gates in the kernel's precision
    ido, go = O6.route_from_logits(z[rows], K)
    assert np.array_equal(ids[rows], ido)
    np.testing.assert_allclose(gates[rows], go, rtol=4e-6, atol=1e-12)
    # 3. against float64 logits: equal ids except at near ties
    ids64, g64 = O6.route_from_logits(zo, K)
    mismatch = np.any(ids[rows] != ids64, axis=1)
    for r in np.nonzero(mismatch)[0]:
        a, b = set(ids[rows][r].tolist()), set(ids64[r].tolist())
        diff = list(a ^ b) + [i for i, j in zip(ids[rows][r], ids64[r]) if i != j]
        zz = zo[r, diff]
        assert zz.max() - zz.min() <= 2 * bound[r, diff].max(), (r, diff, zz)
    assert mismatch.mean() < 0.01
    np.testing.assert_allclose(gates[rows][~mismatch], g64[~mismatch], rtol=1e-3, atol=1e-7)
    assert ids.min() >= 0 and ids.max() < N
    return ids, gates


@pytest.mark.parametrize("B,D,N,K", [
    (1000, 256, 8, 2),       # TINY router (N=8 -> MMA N=16, zero-filled weight rows), ragged last tile
    (700, 2880, 32, 4),      # G20
    (2000, 2880, 128, 4),    # G120 / F-head style
    (300, 2048, 128, 8),     # Q3
    (400, 7168, 256, 8),     # DeepSeek-V3 shape
    (260, 7168, 384, 8),     # Kimi-K2 shape: two 192-wide MMAs, single TMEM buffer
    (129, 64, 1, 1),         # one expert
    (200, 136, 20, 16),      # K = 16 (largest), D not a multiple of 64
    (1, 512, 500, 3),        # one token, N near the limit
])
def test_router_parity(L, B, D, N, K):
    _check(L, B, D, N, K, seed=1234 + N)


def test_router_g120_full_size(L):
    """BASELINE's G120 per-rank batch (32K tokens, D=2880, N=128, K=4), sampled rows vs O6."""
    _check(L, 32768, 2880, 128, 4, seed=7, sample=1500)


def test_router_ties_and_zero_tokens(L):
    """All-zero tokens: every logit is exactly 0 -> ids 0..K-1, gates exactly 1/N (fp32).
    Duplicated router rows: equal logits, the lower id is listed first."""
    dev = torch.device("cuda:0")
    N, K, D = 16, 4, 128
    x = torch.zeros((300, D), dtype=torch.bfloat16, device=dev)
    w = W.router_weight_torch(N, D, dev)
    ids, gates = L.router(x, w, K)
    assert (ids.cpu() == torch.arange(K, dtype=torch.int32)).all()
    assert (gates.cpu() == 1.0 / N).all()
    x = W.tokens_torch(300, D, 0, dev)
    w2 = w.clone()
    w2[9] = w2[3]                           # experts 3 and 9 always tie
    ids, gates, z = L.router(x, w2, K, logits=True)
    ids, z = ids.cpu().numpy(), z.cpu().numpy()
    assert np.array_equal(z[:, 3], z[:, 9])
    for t in range(300):
        row = ids[t].tolist()
        if 9 in row:
            assert 3 in row and row.index(3) == row.index(9) - 1


def test_router_empty_and_invalid(L):
    dev = torch.device("cuda:0")
    x = torch.zeros((0, 64), dtype=torch.bfloat16, device=dev)
    w = torch.zeros((8, 64), dtype=torch.bfloat16, device=dev)
    ids, gates = L.router(x, w, 2)
    assert ids.shape == (0, 2)
    with pytest.raises(L.LLEPError):
        L.router(torch.zeros((4, 64), dtype=torch.bfloat16, device=dev), w, 9)      # K > N
    with pytest.raises(L.LLEPError):
        L.router(torch.zeros((4, 64), dtype=torch.bfloat16, device=dev),
                 torch.zeros((600, 64), dtype=torch.bfloat16, device=dev), 2)       # N > 512


def test_router_feeds_the_layer(L):
    """Router -> LLEP layer (P=1, TINY shape): the layer output on the router's ids / gates equals
    Eq. 1 (O3) evaluated on those ids / gates."""
    import layer_case as LC
    sh = W.CONFIGS["tiny"]
    dev = torch.device("cuda:0")
    B, D, H, N, K = sh.tokens_per_rank, sh.d_model, sh.d_ff, sh.n_experts, sh.top_k
    x = W.tokens_torch(B, D, 0, dev, 99)
    wr = W.router_weight_torch(N, D, dev, scale=4.0, seed=99)
    ids, gates = L.router(x, wr, K)
    w13, w2 = W.expert_weights_torch(range(N), D, H, dev, 99)
    ctx = L.Context(N, K, D, H, 1, 0, 0, B)
    out = ctx(x, ids, gates, w13, w2)
    torch.cuda.synchronize()
    ref = LC.oracle_rank_output(W.LayerShape(N, K, D, H, B, 1), 0, ids.cpu().numpy(),
                                gates.cpu().numpy(), 99)
    mr, l2 = LC.errors(out.float().cpu().numpy(), ref)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (mr, l2)
