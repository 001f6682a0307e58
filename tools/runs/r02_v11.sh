for c in 4 16 148; do for st in 3 6 12; do ./tools/probes/tma_rate_probe $c $st; done; done > gpurun_out/tma_rate_probe.jsonl 2>&1
cat gpurun_out/tma_rate_probe.jsonl
