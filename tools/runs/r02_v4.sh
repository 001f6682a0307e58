# round 2, pass 4: device epochs + capture-safe llep_moe_layer (CUDA graph) + GPU-issued weight pushes
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_r02_v4.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02_v4.log 2>&1
timeout 600 python -m pytest tests/test_gpu_graph.py -q -x > gpurun_out/pytest_r02_v4_graph.log 2>&1; echo rc=$? >> gpurun_out/pytest_r02_v4_graph.log
tail -30 gpurun_out/pytest_r02_v4_graph.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_r02_v4.log 2>&1; echo rc=$? >> gpurun_out/pytest_r02_v4.log
tail -25 gpurun_out/pytest_r02_v4.log
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_r02_v4.json 2> gpurun_out/bench_r02_v4.err
tail -c 400 gpurun_out/bench_r02_v4.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r02_v4.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["phases_ms_per_step"], d["roofline"]["frac"], d["clocks"], d.get("graph"), d["e2e"]["value"])
PY
