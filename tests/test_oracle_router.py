"""Pins for O6 (oracle/router.py), the router of Eq. 2: closed forms, brute force
over tiny inputs, special cases and invariances -- nothing here re-types the oracle's formulas."""
import itertools
import math

import numpy as np
import pytest

from oracle import router as O6


def test_closed_form_one_hot_router():
    """W_r with column i = c_i · e_{d(i)} gives z_i = c_i · x[d(i)], so s and the top-K follow by hand."""
    x = np.array([[0.5, -1.0, 2.0]])
    # expert 0 reads x[2] (2.0), expert 1 reads x[0] (0.5), expert 2 reads x[1] (-1.0), expert 3 reads x[2]/2
    w_r = np.zeros((3, 4))
    w_r[2, 0], w_r[0, 1], w_r[1, 2], w_r[2, 3] = 1.0, 1.0, 1.0, 0.5
    ids, gates, z = O6.route(x, w_r, 2)
    assert z.tolist() == [[2.0, 0.5, -1.0, 1.0]]
    den = math.exp(2.0) + math.exp(0.5) + math.exp(-1.0) + math.exp(1.0)
    assert ids.tolist() == [[0, 3]]
    assert gates[0, 0] == pytest.approx(math.exp(2.0) / den, rel=1e-15)
    assert gates[0, 1] == pytest.approx(math.exp(1.0) / den, rel=1e-15)


def test_uniform_logits_ties_go_to_lower_ids():
    """All logits equal: s_i = 1/N exactly and the K selected are 0..K-1 in order (R31, R32)."""
    ids, gates = O6.route_from_logits(np.zeros((3, 8)), 3)
    assert ids.tolist() == [[0, 1, 2]] * 3
    assert np.all(gates == 1.0 / 8)


def test_brute_force_top_k_tiny():
    """Every vector over {0,1,2}^5 and every K: the selected set maximises Σ s over all K-subsets,
    is lexicographically smallest among the maximisers, and is listed by (s desc, id asc)."""
    for vals in itertools.product(range(3), repeat=5):
        z = np.array([vals], dtype=np.float64)
        s = O6.softmax(z)[0]
        for K in range(1, 6):
            ids, gates = O6.route_from_logits(z, K)
            sel = sorted(ids[0].tolist())
            best = max(itertools.combinations(range(5), K), key=lambda c: (sum(vals[i] for i in c), [-i for i in c]))
            assert sel == list(best), (vals, K)
            order = sorted(sel, key=lambda i: (-vals[i], i))
            assert ids[0].tolist() == order
            assert np.array_equal(gates[0], s[ids[0]])


def test_softmax_special_values():
    """Two experts: s_0 = 1/(1+e^(z1-z0)) (the logistic function); a huge shift changes nothing."""
    z = np.array([[0.3, -1.2], [1000.3, 998.8]])
    s = O6.softmax(z)
    want = 1.0 / (1.0 + math.exp(-1.5))
    assert s[0, 0] == pytest.approx(want, rel=1e-15) and s[1, 0] == pytest.approx(want, rel=1e-12)
    assert np.all(np.isfinite(s))


def test_k_equals_n_and_k_one():
    rng = np.random.default_rng(3)
    x, w_r = rng.standard_normal((6, 5)), rng.standard_normal((5, 7))
    ids, gates, z = O6.route(x, w_r, 7)
    assert np.allclose(gates.sum(axis=1), 1.0, rtol=0, atol=1e-15)   # K = N: the gates are all of s
    assert all(sorted(r) == list(range(7)) for r in ids.tolist())
    ids1, g1, _ = O6.route(x, w_r, 1)
    assert ids1[:, 0].tolist() == np.argmax(z, axis=1).tolist()     # K = 1: argmax (numpy routine)
    assert np.allclose(g1[:, 0], 1.0 / np.exp(z - z.max(axis=1, keepdims=True)).sum(axis=1), rtol=1e-14)


def test_permutation_equivariance_and_dense_form():
    """Relabelling experts (permuting W_r's columns) relabels the selection; Eq. 2's dense g has
    exactly K non-zeros per token whose values are the softmax entries of the selected experts."""
    rng = np.random.default_rng(5)
    x, w_r = rng.standard_normal((20, 6)), rng.standard_normal((6, 9))
    perm = rng.permutation(9)
    ids, gates, z = O6.route(x, w_r, 3)
    ids_p, gates_p, _ = O6.route(x, w_r[:, perm], 3)
    assert np.array_equal(perm[ids_p], ids)      # continuous random logits: no ties
    assert np.allclose(gates_p, gates, rtol=1e-14, atol=0)  # same values; the softmax sum order differs
    g = O6.dense_gates(ids, gates, 9)
    assert np.all((g != 0).sum(axis=1) == 3)
    s = O6.softmax(z)
    assert np.array_equal(g[g != 0], s[g != 0])
    # every unselected s is <= every selected s (top-K property)
    for t in range(20):
        assert s[t][g[t] == 0].max() <= s[t][g[t] != 0].min()


def test_empty_batch():
    ids, gates, z = O6.route(np.zeros((0, 4)), np.ones((4, 3)), 2)
    assert ids.shape == (0, 2) and gates.shape == (0, 2) and z.shape == (0, 3)
