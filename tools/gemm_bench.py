"""Micro-benchmark of the grouped GEMMs through llep_grouped_gemm (C ABI), A/B over env toggles.

    python tools/gemm_bench.py [--layout g120p1|g120p8|uniform|fgemm] [--iters 20]

Group layouts: g120p1 = G120 at P=1 (1 hot group of 124518 rows + 127 groups of 51-52 rows),
g120p8 = one LLEP device at P=8 (a 124464-row spilled chunk + 16 native groups of ~413 rows),
fgemm = the paper's F-gemm shape (65536 tokens over E experts)."""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_17111_b200 import llep as L  # noqa: E402


def layout(name):
    if name == "g120p1":
        return [124518] + [52] * 77 + [51] * 50
    if name == "g120p8":
        return [124464] + [413] * 16
    if name == "g120p8r0":      # the planner's critical rank at G120 P=8 95 %/1 (r02_p8_layout_gemm.jsonl)
        return [124832] + [416] * 15
    if name == "q3p1":          # Q3 at P=1: D=2048, H=768 (use --D 2048 --H 768)
        return [498074] + [207] * 28 + [206] * 99
    if name == "dense":         # one group with G120-P1's real rows (no cold experts)
        return [131072]
    if name == "hot":           # G120-P1's hot group alone
        return [124518]
    if name == "cold":          # G120-P1's 127 cold groups alone
        return [52] * 77 + [51] * 50
    if name == "dsv3p1":        # DeepSeek-V3 shape at P=1 (use --D 7168 --H 2048): hot + 255 cold of ~26 rows
        return [124518] + [26] * 83 + [25] * 172
    if name == "dsv3cold":
        return [26] * 83 + [25] * 172
    if name == "uniform":
        return [1024] * 128
    if name.startswith("fgemm"):
        E = int(name[5:] or 16)
        return [65536 // E] * E
    raise ValueError(name)


def groups_of(sizes, n_weights, ra=128):
    g, rb = [], 0
    for i, n in enumerate(sizes):
        g.append((i % n_weights, rb, n))
        rb += (n + ra - 1) // ra * ra
    return g, rb


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default="g120p1")
    ap.add_argument("--D", type=int, default=2880)
    ap.add_argument("--H", type=int, default=2880)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--variants", default="cta1,cta2")
    ap.add_argument("--burst", action="store_true",
                    help="MEASURED_PEAKS' method: best of --iters single launches, each after 0.5 s idle + a 2 ms spin, "
                         "with cuBLAS timed the same way on 8192^3 and on a dense GEMM of the same FLOPs")
    args = ap.parse_args()
    if args.burst:
        return burst(args)
    D, H = args.D, args.H
    sizes = layout(args.layout)
    E = len(sizes)
    groups1, rows1 = groups_of(sizes, E, 128)
    groups2, rows = groups_of(sizes, E, int(os.environ.get("GB_RA", "256")))
    x = torch.randn(rows, D, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(E, 2 * H, D, device="cuda") / D ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(E, D, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
    act = torch.empty(rows, H, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(rows, D, device="cuda", dtype=torch.bfloat16)
    gate = torch.rand(rows, device="cuda")
    real = sum(sizes)
    res = {}
    for variant in args.variants.split(",") * 2:
        if variant == "group_order":
            os.environ["LLEP_GEMM_GROUP_ORDER"] = "1"
        else:
            os.environ.pop("LLEP_GEMM_GROUP_ORDER", None)
        pair = variant == "cta2"
        groups = groups2 if pair else groups1
        for mode in (0, 1):
            ts = []
            for it in range(args.iters + 3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if mode == 0:
                    L.grouped_gemm(0, x, w13, groups, H, out=act, pair=pair)
                else:
                    L.grouped_gemm(1, act, w2, groups, D, gate=gate, out=y, pair=pair)
                e1.record()
                torch.cuda.synchronize()
                if it >= 3:
                    ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            flops = (4 if mode == 0 else 2) * D * H * real
            res.setdefault((variant, mode), []).append(ms)
            print(f"{args.layout:8s} {variant:12s} gemm{mode + 1}: {ms:7.3f} ms  {flops / ms / 1e9:7.1f} TFLOP/s")
    return res


def _best_idle(fn, n):
    import json  # noqa: F401
    import time
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        time.sleep(0.5)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(4_000_000)   # ~2 ms spin: the host enqueues the launch (and its argument copies)
        e0.record()                    # while the GPU is busy, so e0 -> e1 is the kernel alone
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), statistics.median(ts)


def burst(args):
    import json
    D, H = args.D, args.H
    sizes = layout(args.layout)
    E = len(sizes)
    groups, rows = groups_of(sizes, E, 256)
    real = sum(sizes)
    x = torch.randn(rows, D, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(E, 2 * H, D, device="cuda") / D ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(E, D, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
    act = torch.empty(rows, H, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(rows, D, device="cuda", dtype=torch.bfloat16)
    gate = torch.rand(rows, device="cuda")
    a = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
    b = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
    best, med = _best_idle(lambda: a @ b, args.iters)
    cub = 2 * 8192 ** 3 / best / 1e9
    out = {"layout": args.layout, "rows": real, "groups": E, "method": f"best of {args.iters} launches, each after 0.5 s idle and a ~2 ms spin kernel (host enqueue hidden)",
           "cublas_8192": {"ms": best, "tflops": cub, "median_tflops": 2 * 8192 ** 3 / med / 1e9}}
    xd = torch.randn(real, D, device="cuda").to(torch.bfloat16)
    wd = torch.randn(D, 2 * H, device="cuda").to(torch.bfloat16)
    best, med = _best_idle(lambda: xd @ wd, args.iters)
    out["cublas_dense_same_flops_gemm1"] = {"ms": best, "tflops": 4 * D * H * real / best / 1e9}
    for mode in (0, 1):
        if mode == 0:
            fn = lambda: L.grouped_gemm(0, x, w13, groups, H, out=act, pair=True)  # noqa: E731
        else:
            fn = lambda: L.grouped_gemm(1, act, w2, groups, D, gate=gate, out=y, pair=True)  # noqa: E731
        best, med = _best_idle(fn, args.iters)
        tf = (4 if mode == 0 else 2) * D * H * real / best / 1e9
        out[f"gemm{mode + 1}"] = {"ms": best, "tflops": tf, "median_ms": med, "frac_of_cublas_8192_same_method": tf / cub}
    print(json.dumps(out))
    return out


if __name__ == "__main__":
    main()
