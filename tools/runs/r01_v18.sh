timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k gemm_bwd > gpurun_out/pytest_v18.log 2>&1; echo rc=$? >> gpurun_out/pytest_v18.log
timeout 600 python -m pytest tests/test_gpu_backward.py tests/test_gpu_fuzz.py -x -q >> gpurun_out/pytest_v18.log 2>&1; echo rc=$? >> gpurun_out/pytest_v18.log
timeout 300 python tools/fwd_ab.py LLEP_BWD_SWAP 0 1 --train --reps 2 --secs 4 > gpurun_out/bswap_ab18.jsonl 2>&1
timeout 300 python tools/fwd_ab.py LLEP_BWD_SWAP 1 0 --train --reps 2 --secs 4 >> gpurun_out/bswap_ab18.jsonl 2>&1
timeout 300 python tools/fwd_ab.py LLEP_BWD_SWAP 0 1 --train --reps 2 --secs 4 --config dsv3 >> gpurun_out/bswap_ab18.jsonl 2>&1
grep -E "passed|failed|rc=" gpurun_out/pytest_v18.log; cat gpurun_out/bswap_ab18.jsonl | cut -c1-330
