timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_v14.log 2>&1; echo rc=$? >> gpurun_out/pytest_v14.log
timeout 300 python tools/fwd_ab.py LLEP_GEMM_SWAP 0 1 --secs 3 > gpurun_out/swap_ab14.jsonl 2>&1
timeout 300 python tools/fwd_ab.py LLEP_GEMM_SWAP 1 0 --secs 3 >> gpurun_out/swap_ab14.jsonl 2>&1
timeout 300 python tools/fwd_ab.py LLEP_GEMM_SWAP 0 1 --secs 3 --config dsv3 >> gpurun_out/swap_ab14.jsonl 2>&1
timeout 300 python tools/fwd_ab.py LLEP_GEMM_SWAP 0 1 --secs 3 --config q3 >> gpurun_out/swap_ab14.jsonl 2>&1
timeout 300 python tools/fwd_ab.py LLEP_GEMM_SWAP 0 1 --secs 3 --hot 0 >> gpurun_out/swap_ab14.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_v14.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_v14.log
grep -E "passed|failed|rc=|Error|assert" gpurun_out/pytest_v14.log | head; cat gpurun_out/swap_ab14.jsonl | cut -c1-330; tail -3 gpurun_out/pytest_gpu_v14.log
