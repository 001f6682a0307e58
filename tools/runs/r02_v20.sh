LLEP_BENCH_SHARE_GPU=1 LLEP_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 \
  --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 8 --config q3 --mem-cap-gb 10 --steps 2 --warmup 3 \
  --no-backward --no-e2e --no-distinct --no-cpu-baseline > gpurun_out/bench_q3_p8_cap.json 2> gpurun_out/bench_q3_p8_cap.err
echo rc=$?
tail -c 1500 gpurun_out/bench_q3_p8_cap.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q3_p8_cap.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step", "peak_gb_per_gpu", "ep", "plan", "llep_equals_ep_bitwise")}, d.get("graph"))
PY
