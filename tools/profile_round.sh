#!/bin/bash
# Profile capture for one round (run under gpurun): the bench line, a launch list of the library's
# kernels (share of a step), one ncu --set full capture per hot kernel.  usage: tools/profile_round.sh r01
R=${1:-r01}
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_${R}.txt
timeout 900 python bench.py > gpurun_out/bench_${R}.json 2> gpurun_out/bench_${R}.err
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:llep \
    --csv --log-file gpurun_out/launches_${R}.csv $B > gpurun_out/launch_bench_${R}.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:grouped_gemm -s 16 -c 2 -o gpurun_out/prof_gemm_${R} $B --no-backward > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:"dispatch|combine|planner|layout" -s 24 -c 4 -o gpurun_out/prof_route_${R} $B --no-backward > /dev/null 2>&1
ncu --set full --clock-control none --kernel-name-base mangled \
    -k regex:gemm_bwd -s 4 -c 4 -o gpurun_out/prof_bwd_${R} $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:router -s 3 -c 1 -o gpurun_out/prof_router_${R} python tools/router_bench.py g120 > /dev/null 2>&1
ls -la gpurun_out/
