M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum
for v in default fake_skip_b fake_skip_a; do
  if [ $v = default ]; then unset LLEP_LIB; else export LLEP_LIB=paper_2601_17111_b200/_ab/$v/libllep.so; fi
  timeout 300 ncu --metrics $M --clock-control none -k regex:grouped_gemm -c 2 --csv python tools/gemm_bench.py --layout hot --variants cta2 --iters 1 > gpurun_out/ingest_$v.csv 2>&1
done
