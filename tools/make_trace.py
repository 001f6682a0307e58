"""Write a SPEC-format trace of per-device per-expert slot counts whose imbalance changes
per batch, as Fig. 2 observes for gpt-oss-20b: one record per scenario, every device's
row drawn as the exact slot multiset of that scenario (synth.slot_counts), hot experts rotated per
record so the hot device changes.

    python tools/make_trace.py --config g120 --world 8 --out tools/traces/g120_mix.csv
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import workload as W  # noqa: E402

SCENARIOS = [(95, 1), (80, 4), (50, 16), (30, 1), (None, 0), (95, 4)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="g120")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    sh = W.CONFIGS[a.config]
    N, S = sh.n_experts, sh.tokens_per_rank * sh.top_k
    with open(a.out, "w") as f:
        f.write(f"# {a.config}: N={N}, K={sh.top_k}, {sh.tokens_per_rank} tokens per device, P={a.world}; "
                f"per-device counts, device-major; scenarios {SCENARIOS}\n")
        for r, (hot, nhot) in enumerate(SCENARIOS):
            c = np.roll(W.slot_counts(N, S, hot, min(nhot, N - 1) if hot else 0), r * (N // a.world) // 2)
            f.write(f"{W.scenario_name(hot, nhot)}_r{r}," + ",".join(str(int(v)) for v in np.tile(c, a.world)) + "\n")


if __name__ == "__main__":
    main()
