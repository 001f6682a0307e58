# round 2 final validation + profile pass (the code at HEAD)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_r02_final.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r02_final.log 2>&1; tail -1 gpurun_out/smoke_r02_final.log
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_r02_final.log 2>&1; echo rc=$? >> gpurun_out/pytest_r02_final.log
tail -3 gpurun_out/pytest_r02_final.log
timeout 900 python bench.py > gpurun_out/bench_r02_final.json 2> gpurun_out/bench_r02_final.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_r02_final.json 2> gpurun_out/bench_ref_r02_final.err
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-emulation --no-distinct"
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:llep \
    --csv --log-file gpurun_out/launches_r02_final.csv $B > gpurun_out/launch_bench_r02_final.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:grouped_gemm -s 16 -c 2 -o gpurun_out/prof_gemm_r02_final $B --no-backward > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:"dispatch|combine|planner|layout" -s 24 -c 4 -o gpurun_out/prof_route_r02_final $B --no-backward > /dev/null 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_r02_final.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'], d['graph'].get('ms_per_step'), d['e2e']['value'], d.get('p8_critical_rank_emulation',{}).get('gemm_speedup'))"
ls gpurun_out/*final*
