LLEP_WGRAD_DIRECT=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_backward.py -x -q > gpurun_out/pytest_v10.log 2>&1; echo rc=$? >> gpurun_out/pytest_v10.log
for d in 0 1 0 1; do echo "== direct=$d"; LLEP_WGRAD_DIRECT=$d python tools/wgrad_bench.py small 5760 2880; LLEP_WGRAD_DIRECT=$d python tools/wgrad_bench.py hot 5760 2880; done > gpurun_out/wgrad_ab10.txt 2>&1
python tools/fwd_ab.py LLEP_WGRAD_DIRECT 0 1 --train --reps 2 --secs 4 >> gpurun_out/wgrad_ab10.txt 2>&1
python tools/fwd_ab.py LLEP_WGRAD_DIRECT 1 0 --train --reps 2 --secs 4 >> gpurun_out/wgrad_ab10.txt 2>&1
python tools/fwd_ab.py LLEP_WGRAD_DIRECT 0 1 --train --reps 2 --secs 4 --config q3 >> gpurun_out/wgrad_ab10.txt 2>&1
tail -2 gpurun_out/pytest_v10.log; cat gpurun_out/wgrad_ab10.txt | cut -c1-300
