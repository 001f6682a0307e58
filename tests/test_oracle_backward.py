"""Pins for O5 (oracle/backward.py): central finite differences of the forward definition (O3),
special cases, and the simulated-device LLEP backward with weight-gradient return."""
import numpy as np
import pytest

from oracle import backward as O5
from oracle import layer as O3


def _problem(seed, T=4, K=2, D=5, H=4, N=3):
    rng = np.random.default_rng(seed)
    Ws = {e: (rng.standard_normal((H, D)) / np.sqrt(D), rng.standard_normal((H, D)) / np.sqrt(D),
              rng.standard_normal((D, H)) / np.sqrt(H)) for e in range(N)}
    x = rng.standard_normal((T, D))
    ids = rng.integers(0, N, (T, K))
    ids[0, :] = 1  # a duplicate-id token
    g = rng.random((T, K))
    dout = rng.standard_normal((T, D))
    return Ws, x, ids, g, dout


def _loss(x, ids, g, Ws, dout):
    return float(np.sum(O3.moe_forward(x, ids, g, Ws.get) * dout))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_finite_differences(seed):
    """Every gradient O5 returns equals the central difference of L = Σ <out, dout> computed
    with the FORWARD oracle O3 (independent code path), ε = 1e-6, within 1e-6 relative."""
    Ws, x, ids, g, dout = _problem(seed)
    dx, dg, dW = O5.moe_backward(x, ids, g, dout, Ws.get)
    eps = 1e-6

    def check(analytic, arr, set_fn):
        flat = arr.reshape(-1)
        for i in range(flat.size):
            old = flat[i]
            flat[i] = old + eps
            lp = set_fn()
            flat[i] = old - eps
            lm = set_fn()
            flat[i] = old
            fd = (lp - lm) / (2 * eps)
            assert abs(fd - analytic.reshape(-1)[i]) <= 1e-6 * max(1.0, abs(fd)), (i, fd, analytic.reshape(-1)[i])

    check(dx, x, lambda: _loss(x, ids, g, Ws, dout))
    check(dg, g, lambda: _loss(x, ids, g, Ws, dout))
    for e, (dwg, dwu, dwd) in dW.items():
        for analytic, arr in zip((dwg, dwu, dwd), Ws[e]):
            check(analytic, arr, lambda: _loss(x, ids, g, Ws, dout))


def test_special_cases():
    Ws, x, ids, g, dout = _problem(5)
    dx, dg, dW = O5.moe_backward(x, ids, g, np.zeros_like(dout), Ws.get)
    assert not dx.any() and not dg.any() and all(not a.any() for w in dW.values() for a in w)
    # an expert never routed to has no gradient entry; gate 0 -> that slot adds nothing to dx / dW
    assert set(dW) == set(np.unique(ids).tolist())
    g0 = g.copy()
    g0[:, 1] = 0.0
    ids1 = ids.copy()
    ids1[:, 1] = ids[:, 0]
    a = O5.moe_backward(x, ids1, g0, dout, Ws.get)
    b = O5.moe_backward(x, ids[:, :1], g0[:, :1], dout, Ws.get)
    np.testing.assert_allclose(a[0], b[0], rtol=1e-14, atol=1e-14)
    # dsilu is the derivative of silu
    z = np.linspace(-6, 6, 25)
    np.testing.assert_allclose(O5.dsilu(z), (O5.silu(z + 1e-6) - O5.silu(z - 1e-6)) / 2e-6, rtol=1e-7, atol=1e-9)


def _sim(rng, P, M, K, B, D, H, hot, m, lam):
    N = P * M
    Ws = {e: (rng.standard_normal((H, D)) / np.sqrt(D), rng.standard_normal((H, D)) / np.sqrt(D),
              rng.standard_normal((D, H)) / np.sqrt(H)) for e in range(N)}
    xs, ids, gs, dos = [], [], [], []
    for p in range(P):
        xs.append(rng.standard_normal((B, D)))
        i = rng.integers(0, N, (B, K))
        i[rng.random((B, K)) < hot] = 0
        ids.append(i)
        gs.append(rng.random((B, K)))
        dos.append(rng.standard_normal((B, D)))
    return N, Ws, xs, ids, gs, dos


@pytest.mark.parametrize("seed", range(6))
def test_llep_backward_equals_dense(seed):
    """Backward under EP and under LLEP (spills, forced chunks, weight-gradient return to the native
    device) equals the dense gradients within 1e-12 (the method is exact)."""
    rng = np.random.default_rng(40 + seed)
    P = [2, 3, 4][seed % 3]
    N, Ws, xs, ids, gs, dos = _sim(rng, P, 1 + seed % 2, 2, 12 + seed, 5, 4, 0.7, [0, 3, 20][seed % 3], 1.0)
    dense = [O5.moe_backward(xs[p], ids[p], gs[p], dos[p], Ws.get) for p in range(P)]
    dW_dense = {}
    for p in range(P):
        for e, w in dense[p][2].items():
            dW_dense[e] = w if e not in dW_dense else tuple(a + b for a, b in zip(dW_dense[e], w))
    for mode in ("ep", "llep"):
        dx, dg, dW, plan = O5.dispatch_combine_backward(xs, ids, gs, dos, Ws.get, N, P, mode=mode,
                                                        min_chunk=[0, 3, 20][seed % 3], lam=1.0)
        if mode == "llep":
            assert plan.transfers, "the spill path must be exercised"
        for p in range(P):
            np.testing.assert_allclose(dx[p], dense[p][0], rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(dg[p], dense[p][1], rtol=1e-12, atol=1e-12)
        assert set(dW) == set(dW_dense)
        for e in dW:
            for a, b in zip(dW[e], dW_dense[e]):
                np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)
