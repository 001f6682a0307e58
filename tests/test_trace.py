"""Row f4 (trace replay): SPEC's trace format -> load matrices -> planner / routing.
CPU only."""
import os

import numpy as np
import pytest

from oracle import planner as O1
from synth import workload as W

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_fig2a_record_ratio():
    """Fig. 2(a): E11 holds 20 % of the load at N=32 -> imbalance ratio 0.20/(1/32) = 6.4
    (SPEC S:509-511), through the trace loader and the oracle's λ-test ratio."""
    recs = W.load_trace(os.path.join(GOLDEN, "trace_fig2a.csv"), 32, world=8)
    assert len(recs) == 1 and recs[0].shape == (8, 32)
    l = recs[0].sum(axis=0)
    assert l.sum() == 4000 and l[11] == 800 and recs[0][1:].sum() == 0   # reduced record -> device 0
    assert O1.imbalance_ratio(l.tolist()) == pytest.approx(6.4, rel=1e-12)
    p = O1.plan(l.tolist(), 8, 1.0, 16, 1.3)
    assert not p.fallback and max(p.assigned) <= p.capacity       # 6.4 ≥ λ: LLEP plans a spill


def test_per_device_records_and_errors(tmp_path):
    f = tmp_path / "t.csv"
    f.write_text("# comment\n\nr0, 1,2,3,4, 5,6,7,8\nr1,0,0,0,4,0,0,0,0\n")
    recs = W.load_trace(str(f), 4, world=2)
    assert [r.tolist() for r in recs] == [[[1, 2, 3, 4], [5, 6, 7, 8]], [[0, 0, 0, 4], [0, 0, 0, 0]]]
    for text, msg in [("r,1,2,x,4\n", ":1: malformed"), ("r,1,-2,3,4\n", ":1: negative"),
                      ("ok,1,2,3,4\nr,1,2,3\n", ":2: 3 counts")]:
        f.write_text(text)
        with pytest.raises(W.TraceError, match=msg):
            W.load_trace(str(f), 4, world=2)
    f.write_text("")
    assert W.load_trace(str(f), 4) == []


def test_routing_from_counts_exact_multiset():
    counts = np.array([5, 0, 3, 8, 0, 0, 2, 2])
    ids = W.routing_from_counts(counts, 4, rank=3)
    assert ids.shape == (5, 4) and ids.dtype == np.int32
    assert np.array_equal(np.bincount(ids.ravel(), minlength=8), counts)
    assert np.array_equal(ids, W.routing_from_counts(counts, 4, rank=3))       # deterministic
    with pytest.raises(W.TraceError):
        W.routing_from_counts(np.array([1, 2]), 2, 0)
