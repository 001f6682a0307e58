LLEP_LIB=build/ab/libllep_fk3.so timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k grouped > gpurun_out/pytest_v19.log 2>&1; echo rc=$? >> gpurun_out/pytest_v19.log
for lib in paper_2601_17111_b200/libllep.so build/ab/libllep_fk3.so paper_2601_17111_b200/libllep.so build/ab/libllep_fk3.so; do
  echo "== $lib"; LLEP_LIB=$lib timeout 300 python tools/fwd_ab.py LLEP_DUMMY 0 1 --secs 3
done > gpurun_out/fk3_ab19.txt 2>&1
for lib in paper_2601_17111_b200/libllep.so build/ab/libllep_fk3.so; do
  echo "== $lib"; LLEP_LIB=$lib timeout 300 python tools/fwd_ab.py LLEP_DUMMY 0 1 --secs 3 --config q3; LLEP_LIB=$lib timeout 300 python tools/fwd_ab.py LLEP_DUMMY 0 1 --secs 3 --hot 0
done >> gpurun_out/fk3_ab19.txt 2>&1
grep -E "passed|failed|rc=" gpurun_out/pytest_v19.log; cat gpurun_out/fk3_ab19.txt | cut -c1-250
