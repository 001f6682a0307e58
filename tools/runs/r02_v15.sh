timeout 900 ncu --set full --import-source on --clock-control none -k regex:grouped_gemm_2cta -s 13 -c 1 -o gpurun_out/prof_q3_gemm2 python bench.py --config q3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-distinct --no-backward > gpurun_out/prof_q3_gemm2.log 2>&1
ncu -i gpurun_out/prof_q3_gemm2.ncu-rep --page details --csv > gpurun_out/prof_q3_gemm2_details.csv 2>&1
ncu -i gpurun_out/prof_q3_gemm2.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_q3_gemm2_source.csv 2>&1
ls -la gpurun_out/prof_q3_gemm2*
