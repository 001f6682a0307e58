timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_backward.py -x -q > gpurun_out/pytest_v23.log 2>&1; echo rc=$? >> gpurun_out/pytest_v23.log
for lib in build/ab/libllep_bal0.so paper_2601_17111_b200/libllep.so build/ab/libllep_bal0.so paper_2601_17111_b200/libllep.so; do
  echo "== $lib"; LLEP_LIB=$lib timeout 120 python tools/wgrad_bench.py both 5760 2880; LLEP_LIB=$lib timeout 300 python tools/fwd_ab.py LLEP_DUMMY 0 1 --train --reps 2 --secs 3
done > gpurun_out/bal_ab23.txt 2>&1
grep -E "passed|failed|rc=" gpurun_out/pytest_v23.log; cat gpurun_out/bal_ab23.txt | cut -c1-250
