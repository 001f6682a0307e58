# round 2 checkpoint: full GPU suite, smoke, default bench (driver-like), reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_r02_v19.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r02_v19.log 2>&1; tail -1 gpurun_out/smoke_r02_v19.log
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_r02_v19.log 2>&1; echo rc=$? >> gpurun_out/pytest_r02_v19.log
tail -4 gpurun_out/pytest_r02_v19.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02_v19.json 2> gpurun_out/bench_r02_v19.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02_v19.json 2> gpurun_out/bench_ref_r02_v19.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r02_v19.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"], d["graph"].get("ms_per_step"), d["e2e"]["value"], d["hbm"])
r = json.loads(open("gpurun_out/bench_ref_r02_v19.json").read().strip().splitlines()[-1])
print(r["value"], r["cpu_baseline"])
PY
