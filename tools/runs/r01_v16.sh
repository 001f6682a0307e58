for lib in build/ab/libllep_rot0.so paper_2601_17111_b200/libllep.so build/ab/libllep_rot0.so paper_2601_17111_b200/libllep.so; do
  echo "== $lib"; LLEP_LIB=$lib timeout 120 python tools/wgrad_bench.py small 5760 2880; LLEP_LIB=$lib timeout 120 python tools/wgrad_bench.py small 2880 2880
done > gpurun_out/wg_rot.txt 2>&1
for lib in build/ab/libllep_rot0.so paper_2601_17111_b200/libllep.so build/ab/libllep_rot0.so paper_2601_17111_b200/libllep.so; do
  echo "== $lib"; LLEP_LIB=$lib timeout 300 python tools/fwd_ab.py LLEP_DUMMY 0 1 --train --reps 2 --secs 3
done >> gpurun_out/wg_rot.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_backward.py -q -x >> gpurun_out/wg_rot.txt 2>&1
ncu --set full --clock-control none --kernel-name-base mangled -k regex:gemm_bwd_pair -s 3 -c 1 -o gpurun_out/prof_wgrad_rot python tools/wgrad_bench.py small 5760 2880 > /dev/null 2>&1
cat gpurun_out/wg_rot.txt | cut -c1-230
