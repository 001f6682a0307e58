"""Summaries of ncu output for profiles/: launch list shares and per-kernel key metrics.

    python tools/ncu_summary.py launches <launches.csv>
    python tools/ncu_summary.py full <report.ncu-rep>
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

UNIT = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}


def short(name):
    m = re.search(r"(grouped_gemm_2cta_kernel|grouped_gemm_kernel)ILi(\d+)ELi(\d)E", name)
    if not m:
        m = re.search(r"(grouped_gemm_2cta_kernel|grouped_gemm_kernel)<(?:\(int\))?(\d+), (?:\(int\))?(\d)[,>]", name)
    if m:
        kind = {"0": "GEMM1+SwiGLU", "1": "GEMM2+gate", "2": "GEMM1 recompute, raw gate/up (backward)", "3": "GEMM1+SwiGLU saving [g|u] (training forward)"}[m.group(3)]
        return f"{m.group(1)}<{m.group(2)},{m.group(3)}> ({kind})"
    m = re.search(r"gemm_bwd_pair_kernelILi(\d)E", name) or re.search(r"gemm_bwd_pair_kernel<(?:\(int\))?(\d)[,>]", name)
    if m:
        return f"gemm_bwd_pair_kernel<{m.group(1)}> ({'dY·W / dGU·W13 (MN-major B)' if m.group(1) == '0' else 'weight gradients (MN-major A, B)'})"
    m = re.search(r"router_kernelILi(\d+)E", name) or re.search(r"router_kernel<(?:\(int\))?(\d+)", name)
    if m:
        return f"router_kernel<K={m.group(1)}> (Eq. 2 logits + softmax top-K)"
    m = re.search(r"gemm_bwd_kernelILi(\d)E", name) or re.search(r"gemm_bwd_kernel<(?:\(int\))?(\d)>", name)
    if m:
        return f"gemm_bwd_kernel<{m.group(1)}> ({'dY·W / dGU·W13 (MN-major B)' if m.group(1) == '0' else 'weight gradients (MN-major A, B)'})"
    m = re.search(r"([a-z_0-9]+_kernel)", name)
    return m.group(1) if m else name[:50]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi:
            agg[short(r[ki])].append(float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1))
    tot = sum(sum(v) for v in agg.values())
    print(f"| kernel | launches | mean us | share of library GPU time |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot * 100:.1f} % |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    want = [("gpu__time_duration.sum", "duration"), ("sm__cycles_elapsed.avg.per_second", "SM clock"),
            ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
            ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
            ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
            ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
            ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("launch__registers_per_thread", "regs"),
            ("launch__grid_size", "grid"), ("launch__cluster_dim_x", "cluster")]
    idx = {w: hdr.index(w) for w, _ in want if w in hdr}
    ki = hdr.index("Kernel Name")
    print("| kernel | " + " | ".join(n for w, n in want if w in idx) + " |")
    print("|---" * (1 + len(idx)) + "|")
    for r in rows[2:]:
        cells = [f"{r[idx[w]]} {units[idx[w]]}".strip() for w, _ in want if w in idx]
        print(f"| {short(r[ki])} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
