# round 2, pass 3: local-row gather (GEMM1 reads this rank's own rows from x with TMA gather4)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_r02_v3.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02_v3.log 2>&1
timeout 600 python -m pytest tests/test_gpu_layer.py -q -x -k "gather or p1_full or empty or g120_p1 or q3_p1 or f3_shapes" > gpurun_out/pytest_r02_v3.log 2>&1; echo rc=$? >> gpurun_out/pytest_r02_v3.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-backward --no-cpu-baseline > gpurun_out/bench_r02_v3.json 2> gpurun_out/bench_r02_v3.err
LLEP_NO_GATHER=1 timeout 600 python bench.py --steps 30 --warmup 5 --no-backward --no-cpu-baseline --no-e2e --no-distinct > gpurun_out/bench_r02_v3_nogather.json 2> gpurun_out/bench_r02_v3_nogather.err
tail -15 gpurun_out/pytest_r02_v3.log; tail -c 400 gpurun_out/bench_r02_v3.err
python - <<'PY'
import json
for f in ("gpurun_out/bench_r02_v3.json", "gpurun_out/bench_r02_v3_nogather.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d["phases_ms_per_step"], d["roofline"]["frac"], d["clocks"])
    except Exception as e:
        print(f, "ERR", e)
PY
