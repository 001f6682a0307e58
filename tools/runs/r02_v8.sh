# round 2, pass 8: graph tests at P=8, emulation test, profile pass of the current build, shared-GPU P=2 bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_r02_v8.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02_v8.log 2>&1
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_emulation.py -q -x > gpurun_out/pytest_r02_v8.log 2>&1; echo rc=$? >> gpurun_out/pytest_r02_v8.log
tail -5 gpurun_out/pytest_r02_v8.log
bash tools/profile_round.sh r02
LLEP_BENCH_SHARE_GPU=1 LLEP_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --steps 5 --warmup 3 --no-backward \
  > gpurun_out/bench_r02_p2share.json 2> gpurun_out/bench_r02_p2share.err
tail -c 300 gpurun_out/bench_r02_p2share.err; head -c 300 gpurun_out/bench_r02_p2share.json
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r02.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["phases_ms_per_step"], d["roofline"]["frac"], d["clocks"], d.get("graph"))
d = json.loads(open("gpurun_out/bench_r02_p2share.json").read().strip().splitlines()[-1])
print("P2share", d["value"], d.get("graph"), d.get("speedup_vs_ep"))
PY
