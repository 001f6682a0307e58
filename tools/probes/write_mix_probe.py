"""HBM bandwidth for the dispatch's traffic mix on this B200: pure writes (fill_), 1:1 copy (copy_), and
1:4 read:write (each 5760-byte row written K=4 times, via torch.repeat_interleave and via index_select with
the G120 dispatch's row order), CUDA events, best of 10.  -> JSON lines."""
import json

import torch


def bw(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return nbytes / best / 1e6, best


B, D, K = 32768, 2880, 4
x = torch.randn(B, D, device="cuda").to(torch.bfloat16)
big = torch.empty(B * K, D, device="cuda", dtype=torch.bfloat16)
src = torch.empty(4 * B, D, device="cuda", dtype=torch.bfloat16)
idx = torch.randperm(B * K, device="cuda") % B          # each token row written K times, scattered
row = B * K * D * 2
for name, fn, nb in [
    ("fill (pure write)", lambda: big.fill_(1.0), row),
    ("copy 1:1", lambda: big.copy_(src), 2 * row),
    ("repeat_interleave 1:4 (contiguous writes)", lambda: torch.repeat_interleave(x, K, dim=0, output_size=B * K), row + B * D * 2),
    ("index_select 1:4 (gather rows, contiguous writes)", lambda: torch.index_select(x, 0, idx, out=big), row + B * D * 2),
    ("index_copy 1:4 (scatter rows)", lambda: big.index_copy_(0, torch.randperm(B * K, device="cuda"), x.repeat(K, 1)), 0),
]:
    if nb == 0:
        continue
    g, ms = bw(fn, nb)
    print(json.dumps({"op": name, "GBps": round(g, 1), "ms": round(ms, 4), "bytes": nb}), flush=True)
