"""Randomised layer shapes on the GPU (P=1) and degenerate multi-rank cases vs the float64 oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import layer_case as LC  # noqa: E402
from synth import workload as W  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_17111_b200 import llep
    return llep


CASES = [  # N, K, D, H, B, hot, nhot
    (1, 1, 8, 8, 5, None, 0),          # single expert, K=1, minimal widths (TMA OOB fill)
    (4, 4, 72, 40, 333, 95, 1),        # K = N, widths not multiples of 64
    (16, 2, 200, 136, 1000, 80, 4),
    (64, 8, 256, 512, 3000, 50, 16),
    (3, 2, 128, 256, 257, 30, 1),      # N not a power of two
    (32, 1, 64, 64, 4096, None, 0),    # balanced, K=1
]


@pytest.mark.parametrize("case", CASES)
def test_fuzz_p1_forward_backward(L, case):
    from oracle import backward as O5
    N, K, D, H, B, hot, nhot = case
    sh = W.LayerShape(N, K, D, H, B, 1)
    seed = 1000 + N + K + D + H
    x, ids, gates, w13, w2, ids_np, g_np = LC.rank_inputs(sh, 0, hot, nhot, seed, "cuda")
    ctx = L.Context(N, K, D, H, 1, 0, 0, B)
    out = ctx(x, ids, gates, w13, w2, min_chunk=0, lam=1.0)
    torch.cuda.synchronize()
    ref = LC.oracle_rank_output(sh, 0, ids_np, g_np, seed)
    mr, l2 = LC.errors(out.float().cpu().numpy().astype(np.float64), ref)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, ("fwd", case, mr, l2)
    # backward
    ctx.enable_backward()
    dout_bits = W.tokens_bits(B, D, 777, seed)
    dout = torch.from_numpy(dout_bits.view(np.int16)).cuda().view(torch.bfloat16)
    plan, _ = ctx.prepare(ids, 1.0, 0, 1.0)
    dx, dg, dw13, dw2 = ctx.backward(x, ids, gates, dout, w13, w2, plan)
    torch.cuda.synchronize()
    ws = LC.OracleWeights(D, H, seed)
    xr = W.bf16_bits_to_f64(W.tokens_bits(B, D, 0, seed))
    rdx, rdg, rdW = O5.moe_backward(xr, ids_np, g_np.astype(np.float64), W.bf16_bits_to_f64(dout_bits), ws)
    mr, l2 = LC.errors(dx.float().cpu().numpy().astype(np.float64), rdx)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, ("dx", case, mr, l2)
    mr, l2 = LC.errors(dg.cpu().numpy().astype(np.float64), rdg)
    assert l2 <= LC.TOL_REL_L2, ("dgates", case, mr, l2)
    for e in range(N):
        if e in rdW:
            for y, r in ((dw13[e, :H], rdW[e][0]), (dw13[e, H:], rdW[e][1]), (dw2[e], rdW[e][2])):
                mr, l2 = LC.errors(y.cpu().numpy().astype(np.float64), r)
                assert l2 <= LC.TOL_REL_L2, ("dW", case, e, mr, l2)
        else:
            assert not dw13[e].any() and not dw2[e].any()
    ctx.close()


def test_multiprocess_empty_rank(L, tmp_path):
    """P=2 where rank 1 routes no tokens (B=0): the exchange, plan and every barrier still complete,
    and rank 0's output matches the oracle."""
    script = os.path.join(tmp_path, "w.py")
    open(script, "w").write(f"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {os.path.dirname(HERE)!r}); sys.path.insert(0, {HERE!r})
import layer_case as LC
from synth import workload as W
from paper_2601_17111_b200 import llep as L
def main(rank):
    dist.init_process_group('gloo', rank=rank, world_size=2)
    torch.cuda.set_device(0)
    sh = W.LayerShape(8, 2, 256, 512, 512, 2)
    x, ids, g, w13, w2, ids_np, g_np = LC.rank_inputs(sh, rank, 95, 1, 5, 'cuda:0')
    B = 512 if rank == 0 else 0
    ctx = L.Context(8, 2, 256, 512, 2, rank, 0, 512)
    out = ctx(x[:B].contiguous(), ids[:B].contiguous(), g[:B].contiguous(), w13, w2, min_chunk=0, lam=1.0)
    torch.cuda.synchronize()
    np.save(os.path.join({str(tmp_path)!r}, f'out{{rank}}.npy'), out.float().cpu().numpy())
    dist.barrier(); ctx.close()
if __name__ == '__main__':
    import torch.multiprocessing as mp
    mp.spawn(main, nprocs=2, join=True)
""")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29911")
    r = subprocess.run([sys.executable, script], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    sh = W.LayerShape(8, 2, 256, 512, 512, 2)
    ids0 = W.routing_ids(sh, 0, 95, 1, 5)
    g0 = W.gate_weights(512, 2, 0, 5)
    ref = LC.oracle_rank_output(sh, 0, ids0, g0, 5)
    out0 = np.load(os.path.join(tmp_path, "out0.npy")).astype(np.float64)
    mr, l2 = LC.errors(out0, ref)
    assert mr <= LC.TOL_MAX_REL and l2 <= LC.TOL_REL_L2, (mr, l2)
    assert np.load(os.path.join(tmp_path, "out1.npy")).shape == (0, 256)
