#!/bin/bash
# Profile capture for one round (run under gpurun): launch list of the library's kernels (share of a
# step) and one ncu --set full capture per hot kernel.  usage: tools/profile_round.sh r01
R=${1:-r01}
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:llep \
    --csv --log-file gpurun_out/launches_${R}.csv $B > gpurun_out/launch_bench_${R}.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:grouped_gemm -s 16 -c 2 -o gpurun_out/prof_gemm_${R} $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:"dispatch|combine|local_rank|planner|layout" -s 30 -c 5 -o gpurun_out/prof_route_${R} $B > /dev/null 2>&1
ls -la gpurun_out/
