# per-pair streaming rate of cold (swapped) tiles vs number of CTA pairs (cold-only G120 layout, GEMM1)
mkdir -p gpurun_out/pairs
for np in 2 4 8 16 37 74; do
  LLEP_GEMM_PAIRS=$np timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:grouped_gemm -c 2 --csv python tools/gemm_bench.py --layout cold --variants cta2 --iters 1 > gpurun_out/pairs/cold_$np.csv 2>&1
done
for np in 8 37 74; do
  LLEP_GEMM_PAIRS=$np timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:grouped_gemm -c 1 --csv python tools/gemm_bench.py --layout hot --variants cta2 --iters 1 > gpurun_out/pairs/hot_$np.csv 2>&1
done
ls gpurun_out/pairs
