# round 2, pass 6: hot / cold / both decomposition of the P=1 grouped GEMMs (standalone entry)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02_v6.log 2>&1
for lay in hot cold g120p1 dense; do timeout 300 python tools/gemm_bench.py --layout $lay --variants cta2 --iters 20; done > gpurun_out/gemm_decomp_g120.txt 2>&1
for lay in hot dsv3cold dsv3p1; do timeout 300 python tools/gemm_bench.py --layout $lay --D 7168 --H 2048 --variants cta2 --iters 10; done > gpurun_out/gemm_decomp_dsv3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:grouped_gemm -c 8 --csv python tools/gemm_bench.py --layout cold --variants cta2 --iters 1 > gpurun_out/ncu_cold.csv 2>&1
cat gpurun_out/gemm_decomp_g120.txt gpurun_out/gemm_decomp_dsv3.txt; grep -v "^==" gpurun_out/ncu_cold.csv | tail -40
