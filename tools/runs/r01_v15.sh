for lib in paper_2601_17111_b200/libllep.so build/ab/libllep_n6.so build/ab/libllep_n8.so paper_2601_17111_b200/libllep.so build/ab/libllep_n6.so build/ab/libllep_n8.so; do
  echo "== $lib"; LLEP_LIB=$lib timeout 120 python tools/wgrad_bench.py small 5760 2880; LLEP_LIB=$lib timeout 120 python tools/wgrad_bench.py both 5760 2880
done > gpurun_out/wg_nstg.txt 2>&1
for lib in paper_2601_17111_b200/libllep.so build/ab/libllep_n6.so build/ab/libllep_n8.so paper_2601_17111_b200/libllep.so build/ab/libllep_n6.so build/ab/libllep_n8.so; do
  echo "== $lib"; LLEP_LIB=$lib timeout 300 python tools/fwd_ab.py LLEP_DUMMY 0 1 --train --reps 2 --secs 3
done >> gpurun_out/wg_nstg.txt 2>&1
LLEP_LIB=build/ab/libllep_n6.so timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k gemm_bwd >> gpurun_out/wg_nstg.txt 2>&1
LLEP_LIB=build/ab/libllep_n8.so timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k gemm_bwd >> gpurun_out/wg_nstg.txt 2>&1
cat gpurun_out/wg_nstg.txt | cut -c1-230
