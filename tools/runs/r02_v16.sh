# A/B: CTA-scope release on the TMEM-empty arrive (default build) vs .release.cluster (v9 lib)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02_v16.log 2>&1
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for v in new old; do
  if [ $v = old ]; then export LLEP_LIB=paper_2601_17111_b200/_ab/v9/libllep.so; else unset LLEP_LIB; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm_2cta -s 12 -c 2 --csv python bench.py --config q3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-distinct --no-backward > gpurun_out/ab16_q3_$v.csv 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:grouped_gemm_2cta -s 12 -c 2 --csv python bench.py --config g120 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-distinct --no-backward > gpurun_out/ab16_g120_$v.csv 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:router -c 2 --csv python tools/router_bench.py g120 > gpurun_out/ab16_router_$v.csv 2>&1
done
unset LLEP_LIB
for c in g120 q3 fhead; do timeout 600 python tools/fwd_ab.py LLEP_NOOP 0 1 --config $c --secs 3; done > gpurun_out/ab16_fwd.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_router.py tests/test_gpu_backward.py -q -x > gpurun_out/pytest_v16.log 2>&1; tail -3 gpurun_out/pytest_v16.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-backward --no-cpu-baseline --no-distinct > gpurun_out/bench_v16.json 2>gpurun_out/bench_v16.err
LLEP_LIB=paper_2601_17111_b200/_ab/v9/libllep.so timeout 600 python bench.py --steps 30 --warmup 5 --no-backward --no-cpu-baseline --no-distinct > gpurun_out/bench_v16_old.json 2>gpurun_out/bench_v16_old.err
python - <<'PY'
import json
for f in ("gpurun_out/bench_v16.json", "gpurun_out/bench_v16_old.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["ms_per_step"], d["phases_ms_per_step"]["gemm1"], d["phases_ms_per_step"]["gemm2"], d["clocks"]["sm_mhz"])
PY
