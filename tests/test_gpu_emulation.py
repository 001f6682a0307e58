"""GEMM-only critical-rank bound on one B200, NOT the north-star metric: at the G120
layer, P=8, 95 % of slots into one expert, the most loaded rank's grouped GEMM1 + GEMM2 under LLEP run
>= 3x faster than under standard EP on the same kernels (the compute bound is 7.65x), also after adding
each arm's MODELLED NVLink time (dispatch + combine rows and the weight broadcast at 900 GB/s per
direction, tools/emulate_p8.link_seconds).  Dispatch, combine and the weight broadcast are not executed
here; the north-star ratio needs an 8-GPU run (bench.py --gpus 8)."""
import os
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.fixture(scope="module")
def E():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import emulate_p8
    return emulate_p8


def test_critical_rank_gemms_llep_3x_ep_g120_p8_layout(E):
    from synth import workload as W
    from paper_2601_17111_b200 import llep as L
    P = 8
    base = W.CONFIGS["g120"]
    sh = W.LayerShape(base.n_experts, base.top_k, base.d_model, base.d_ff, base.tokens_per_rank, P)
    M = sh.experts_per_rank
    cnt = W.slot_counts(sh.n_experts, sh.tokens_per_rank * sh.top_k, 95, 1)
    loads = (cnt * P).tolist()
    ms = {}
    rows = {}
    link = {}
    for mode in ("ep", "llep"):
        plan = L.plan_host(loads, P, 1.0, 1024, 1.3, ep=(mode == "ep"))
        per_rank = [sum(E.rank_groups(plan, r, M)) for r in range(P)]
        crit = max(range(P), key=lambda r: per_rank[r])
        g = E.Gemms(E.rank_groups(plan, crit, M), sh.d_model, sh.d_ff)
        g.run_ms()
        ms[mode] = min(g.run_ms() for _ in range(3))
        rows[mode] = per_rank[crit]
        link[mode] = E.link_seconds(plan, cnt, sh.d_model, sh.d_ff, M, P) * 1e3
        del g
        torch.cuda.empty_cache()
    assert rows["llep"] == sh.tokens_per_rank * sh.top_k          # every rank at capacity
    assert rows["ep"] / rows["llep"] > 7.6                         # the 7.65x compute bound
    assert ms["ep"] / ms["llep"] >= 3.0, ms
    assert (ms["ep"] + link["ep"]) / (ms["llep"] + link["llep"]) >= 3.0, (ms, link)
