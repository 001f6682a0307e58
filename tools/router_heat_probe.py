"""Router timing on an idle GPU vs right after ~3 s of back-to-back layer steps (is the in-bench router
time a clock effect?).  python tools/router_heat_probe.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2601_17111_b200 import llep as L  # noqa: E402
from synth import workload as W  # noqa: E402

sh = W.CONFIGS["g120"]
shape = W.LayerShape(sh.n_experts, sh.top_k, sh.d_model, sh.d_ff, sh.tokens_per_rank, 1)
x = W.tokens_torch(shape.tokens_per_rank, shape.d_model, 0, "cuda:0")
print("idle", round(bench.run_router(L, shape, x, 20, 3)["ms_per_call"] * 1e3, 1), "us", flush=True)
ids = torch.from_numpy(W.routing_ids(shape, 0, 95, 1, 1)).cuda()
g = torch.from_numpy(W.gate_weights(shape.tokens_per_rank, shape.top_k, 0, 1)).cuda()
w13, w2 = W.expert_weights_torch(range(shape.n_experts), shape.d_model, shape.d_ff, "cuda:0")
ctx = L.Context(shape.n_experts, shape.top_k, shape.d_model, shape.d_ff, 1, 0, 0, shape.tokens_per_rank)
out = torch.empty_like(x)
for load_s in (0.5, 3.0):
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < load_s:
        ctx(x, ids, g, w13, w2, out=out)
        torch.cuda.synchronize()
    print(f"after {load_s} s of layer steps", round(bench.run_router(L, shape, x, 20, 3)["ms_per_call"] * 1e3, 1), "us",
          flush=True)
    time.sleep(2.0)
    print("after 2 s idle", round(bench.run_router(L, shape, x, 20, 3)["ms_per_call"] * 1e3, 1), "us", flush=True)
