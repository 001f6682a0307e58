timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_fuzz.py -x -q -k "not g120_p8 and not large_layer" > gpurun_out/pytest_v17.log 2>&1; echo rc=$? >> gpurun_out/pytest_v17.log
timeout 600 python -m pytest tests/test_gpu_backward.py -x -q >> gpurun_out/pytest_v17.log 2>&1; echo rc=$? >> gpurun_out/pytest_v17.log
for lib in build/ab/libllep_swk2.so paper_2601_17111_b200/libllep.so build/ab/libllep_swk2.so paper_2601_17111_b200/libllep.so; do
  echo "== $lib"; LLEP_LIB=$lib timeout 300 python tools/fwd_ab.py LLEP_GEMM_SWAP 0 1 --secs 3
done > gpurun_out/swk_ab17.txt 2>&1
for lib in build/ab/libllep_swk2.so paper_2601_17111_b200/libllep.so; do
  echo "== $lib"; LLEP_LIB=$lib timeout 300 python tools/fwd_ab.py LLEP_GEMM_SWAP 0 1 --secs 3 --config dsv3
done >> gpurun_out/swk_ab17.txt 2>&1
grep -E "passed|failed|rc=" gpurun_out/pytest_v17.log; cat gpurun_out/swk_ab17.txt | cut -c1-330
