# round 2, pass 9: chunk-aligned token order (R11') on the device: full GPU suite + bench + P=2 shared dry run
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02_v9.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_r02_v9.log 2>&1; echo rc=$? >> gpurun_out/pytest_r02_v9.log
tail -20 gpurun_out/pytest_r02_v9.log
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_r02_v9.json 2> gpurun_out/bench_r02_v9.err
LLEP_BENCH_SHARE_GPU=1 LLEP_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --steps 5 --warmup 3 --no-backward --no-e2e \
  > gpurun_out/bench_r02_v9_p2share.json 2> gpurun_out/bench_r02_v9_p2share.err
tail -c 300 gpurun_out/bench_r02_v9.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r02_v9.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["phases_ms_per_step"], d["roofline"]["frac"], d["clocks"], d["graph"]["ms_per_step"], d["e2e"]["value"])
d = json.loads(open("gpurun_out/bench_r02_v9_p2share.json").read().strip().splitlines()[-1])
print("P2share", d["nvlink"]["llep"], d["roofline"]["layer"])
PY
