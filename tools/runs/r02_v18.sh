M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"gemm_bwd|split_reduce" -c 12 --csv python tools/wgrad_bench.py p8 5760 2880 > gpurun_out/ncu_wgrad_p8.csv 2>&1
grep -v "^==" gpurun_out/ncu_wgrad_p8.csv | tail -40 | cut -d, -f5,13-15
