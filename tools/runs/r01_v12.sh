timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm_bwd" > gpurun_out/pytest_v12.log 2>&1; echo rc=$? >> gpurun_out/pytest_v12.log
timeout 600 python -m pytest tests/test_gpu_backward.py -x -q >> gpurun_out/pytest_v12.log 2>&1; echo rc=$? >> gpurun_out/pytest_v12.log
for d in 0 1 0 1; do echo "== interleave=$d"; LLEP_WGRAD_INTERLEAVE=$d timeout 120 python tools/wgrad_bench.py both 5760 2880; LLEP_WGRAD_INTERLEAVE=$d timeout 120 python tools/wgrad_bench.py both 2880 2880; done > gpurun_out/wgrad_ab12.txt 2>&1
timeout 300 python tools/fwd_ab.py LLEP_WGRAD_INTERLEAVE 0 1 --train --reps 2 --secs 4 >> gpurun_out/wgrad_ab12.txt 2>&1
timeout 300 python tools/fwd_ab.py LLEP_WGRAD_INTERLEAVE 1 0 --train --reps 2 --secs 4 >> gpurun_out/wgrad_ab12.txt 2>&1
timeout 300 python tools/fwd_ab.py LLEP_WGRAD_INTERLEAVE 0 1 --train --reps 2 --secs 4 --config q3 >> gpurun_out/wgrad_ab12.txt 2>&1
grep -E "passed|failed|rc=" gpurun_out/pytest_v12.log; cat gpurun_out/wgrad_ab12.txt | cut -c1-300
