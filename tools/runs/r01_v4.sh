python tools/fwd_ab.py LLEP_GEMM_PREFETCH 0 1 > gpurun_out/fwd_ab_pf.jsonl 2>&1
python tools/fwd_ab.py LLEP_GEMM_PREFETCH 0 1 --hot 0 >> gpurun_out/fwd_ab_pf.jsonl 2>&1
python tools/fwd_ab.py LLEP_GEMM_PREFETCH 0 1 --config q3 >> gpurun_out/fwd_ab_pf.jsonl 2>&1
python tools/fwd_ab.py LLEP_GEMM_PREFETCH 0 1 --config dsv3 --secs 4 >> gpurun_out/fwd_ab_pf.jsonl 2>&1
python tools/fwd_ab.py LLEP_GEMM_PREFETCH 1 0 >> gpurun_out/fwd_ab_pf.jsonl 2>&1
cat gpurun_out/fwd_ab_pf.jsonl
