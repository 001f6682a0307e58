"""Small end-to-end driver for compute-sanitizer (memcheck / synccheck): tiny layer at P=1 through the
two-call path, the capture-safe layer call (direct and replayed from a CUDA graph), forward_train +
backward from the saved pre-activations, and the router; each result checked against the previous.

    compute-sanitizer --tool memcheck python tools/sanitize_layer.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_17111_b200 import llep as L  # noqa: E402
from synth import workload as W  # noqa: E402


def main():
    sh = W.LayerShape(8, 2, 256, 512, 1024, 1)
    x = W.tokens_torch(1024, 256, 0, "cuda", 3)
    ids = torch.from_numpy(W.routing_ids(sh, 0, 95, 1, 3)).cuda()
    g = torch.from_numpy(W.gate_weights(1024, 2, 0, 3)).cuda()
    w13, w2 = W.expert_weights_torch(range(8), 256, 512, "cuda", 3)
    ctx = L.Context(8, 2, 256, 512, 1, 0, 0, 1024)
    ref = ctx(x, ids, g, w13, w2).clone()
    assert torch.equal(ctx.layer(x, ids, g, w13, w2), ref)
    out = torch.empty_like(x)
    plan = torch.empty(L.plan_bytes(8, 1), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ctx.layer(x, ids, g, w13, w2, plan_out=plan, out=out)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ctx.layer(x, ids, g, w13, w2, plan_out=plan, out=out)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    ctx.enable_backward()
    p, _ = ctx.prepare(ids)
    dout = W.tokens_torch(1024, 256, 7, "cuda", 3)
    o2, gu = ctx.forward_train(x, ids, g, w13, w2, p)
    a = ctx.backward(x, ids, g, dout, w13, w2, p)
    b = ctx.backward(x, ids, g, dout, w13, w2, p, gu=gu)
    torch.cuda.synchronize()
    assert torch.equal(o2, ref) and all(torch.equal(u, v) for u, v in zip(a, b))
    wr = W.router_weight_torch(8, 256, "cuda", seed=3)
    L.router(x, wr, 2)
    ctx.check()
    torch.cuda.synchronize()
    del graph
    ctx.close()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
