timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_backward.py -x -q > gpurun_out/pytest_v9.log 2>&1; echo rc=$? >> gpurun_out/pytest_v9.log
for lib in build/ab/libllep_old.so paper_2601_17111_b200/libllep.so build/ab/libllep_old.so paper_2601_17111_b200/libllep.so; do
  echo "== $lib"; LLEP_LIB=$lib python tools/wgrad_bench.py small 5760 2880; LLEP_LIB=$lib python tools/wgrad_bench.py both 5760 2880; LLEP_LIB=$lib python tools/wgrad_bench.py small 2880 2880
done > gpurun_out/wgrad_ab9.txt 2>&1
for lib in build/ab/libllep_old.so paper_2601_17111_b200/libllep.so build/ab/libllep_old.so paper_2601_17111_b200/libllep.so; do
  echo "== $lib"; LLEP_LIB=$lib python tools/fwd_ab.py LLEP_DUMMY 0 1 --train --reps 2 --secs 3
done >> gpurun_out/wgrad_ab9.txt 2>&1
tail -2 gpurun_out/pytest_v9.log; cat gpurun_out/wgrad_ab9.txt | cut -c1-250
