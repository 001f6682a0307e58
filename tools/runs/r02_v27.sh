# P=8 rehearsal of the multi-rank bench (8 processes sharing the GPU; times meaningless): every code path
LLEP_BENCH_SHARE_GPU=1 LLEP_BENCH_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 \
  --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 8 --steps 3 --warmup 3 --no-backward \
  > gpurun_out/bench_p8_rehearsal.json 2> gpurun_out/bench_p8_rehearsal.err
echo rc=$?
tail -c 800 gpurun_out/bench_p8_rehearsal.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_p8_rehearsal.json').read().strip().splitlines()[-1]); print({k: d.get(k) for k in ('value','n_gpus','speedup_vs_ep','peak_gb_per_gpu','plan','llep_equals_ep_bitwise')}); print(d['nvlink']['llep']); print(d['ep']); print(d.get('graph')); print(d.get('e2e'))"
