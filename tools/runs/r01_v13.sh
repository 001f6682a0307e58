timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm_bwd" > gpurun_out/pytest_v13.log 2>&1; echo rc=$? >> gpurun_out/pytest_v13.log
timeout 600 python -m pytest tests/test_gpu_backward.py -x -q >> gpurun_out/pytest_v13.log 2>&1; echo rc=$? >> gpurun_out/pytest_v13.log
for lib in build/ab/libllep_ksub1.so paper_2601_17111_b200/libllep.so build/ab/libllep_ksub1.so paper_2601_17111_b200/libllep.so; do
  echo "== $lib"; LLEP_LIB=$lib timeout 300 python tools/fwd_ab.py LLEP_DUMMY 0 1 --train --reps 2 --secs 3
done > gpurun_out/ksub_ab13.txt 2>&1
for lib in build/ab/libllep_ksub1.so paper_2601_17111_b200/libllep.so build/ab/libllep_ksub1.so paper_2601_17111_b200/libllep.so; do
  echo "== $lib"; LLEP_LIB=$lib timeout 300 python tools/fwd_ab.py LLEP_DUMMY 0 1 --train --reps 2 --secs 3 --config q3
done >> gpurun_out/ksub_ab13.txt 2>&1
ncu --set full --clock-control none --kernel-name-base mangled -k regex:gemm_bwd_pair_kernel -s 2 -c 2 -o gpurun_out/prof_bwd_ksub2 python tools/fwd_ab.py LLEP_DUMMY 0 1 --train --reps 1 --secs 0.1 > /dev/null 2>&1
grep -E "passed|failed|rc=" gpurun_out/pytest_v13.log; cat gpurun_out/ksub_ab13.txt | cut -c1-260
