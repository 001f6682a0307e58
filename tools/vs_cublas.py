"""Our grouped GEMM1 / GEMM2 (C ABI, pair kernels) vs cuBLAS (torch.matmul) on the same FLOPs, timed
back to back in steady state (each >= 150 ms per round, alternating, median), same process.

    python tools/vs_cublas.py [--layouts dense,g120p1,g120p8]
"""
import argparse
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2601_17111_b200 import llep as L  # noqa: E402
from gemm_bench import groups_of, layout  # noqa: E402


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def steady(fns, rounds=3, burst_ms=150.0):
    out = {k: [] for k in fns}
    for k, f in fns.items():
        f()
    torch.cuda.synchronize()
    for _ in range(rounds):
        for k, f in fns.items():
            t0 = time.perf_counter()
            while (time.perf_counter() - t0) * 1e3 < burst_ms or len(out[k]) < 3:
                out[k].append(timed(f))
    return {k: statistics.median(v) for k, v in out.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layouts", default="dense,g120p1,g120p8")
    ap.add_argument("--D", type=int, default=2880)
    ap.add_argument("--H", type=int, default=2880)
    a = ap.parse_args()
    D, H = a.D, a.H
    for name in a.layouts.split(","):
        sizes = [131072] if name == "dense" else layout(name)
        E = len(sizes)
        groups, rows = groups_of(sizes, E, 256)
        real = sum(sizes)
        x = torch.randn(rows, D, device="cuda").to(torch.bfloat16)
        w13 = (torch.randn(E, 2 * H, D, device="cuda") / D ** 0.5).to(torch.bfloat16)
        w2 = (torch.randn(E, D, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
        act = torch.empty(rows, H, device="cuda", dtype=torch.bfloat16)
        y = torch.empty(rows, D, device="cuda", dtype=torch.bfloat16)
        gate = torch.rand(rows, device="cuda")
        xd = torch.randn(real, D, device="cuda").to(torch.bfloat16)
        wd1 = torch.randn(D, 2 * H, device="cuda").to(torch.bfloat16)
        ad = torch.randn(real, H, device="cuda").to(torch.bfloat16)
        wd2 = torch.randn(H, D, device="cuda").to(torch.bfloat16)
        fns = {
            "ours_gemm1": lambda: L.grouped_gemm(0, x, w13, groups, H, out=act, pair=True),
            "cublas_gemm1": lambda: torch.matmul(xd, wd1),
            "ours_gemm2": lambda: L.grouped_gemm(1, act, w2, groups, D, gate=gate, out=y, pair=True),
            "cublas_gemm2": lambda: torch.matmul(ad, wd2),
        }
        ms = steady(fns)
        f1, f2 = 4.0 * real * D * H, 2.0 * real * D * H
        res = {k: (round(v, 3), round((f1 if k.endswith("1") else f2) / (v / 1e3) / 1e12)) for k, v in ms.items()}
        print(name, f"{E} groups, {real} rows:", res,
              "ratio gemm1", round(ms["cublas_gemm1"] / ms["ours_gemm1"], 3),
              "gemm2", round(ms["cublas_gemm2"] / ms["ours_gemm2"], 3), flush=True)
        del x, w13, w2, act, y, gate, xd, wd1, ad, wd2
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
