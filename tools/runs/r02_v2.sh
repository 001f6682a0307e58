# round 2, pass 2: GPU suite timing after the speedups, shared-GPU multi-rank bench dry run, P=8 layout GEMMs + ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_r02_v2.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/pytest_r02_v2.log 2>&1; echo rc=$? >> gpurun_out/pytest_r02_v2.log
LLEP_BENCH_SHARE_GPU=1 LLEP_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --steps 5 --warmup 3 --sweep --no-backward \
  > gpurun_out/bench_r02_v2_p2share.json 2> gpurun_out/bench_r02_v2_p2share.err
for r in 0 1; do timeout 300 python tools/p8_layout_gemm.py --rank $r --iters 30; done > gpurun_out/p8_layout_r02_v2.jsonl 2>&1
timeout 300 python tools/p8_layout_gemm.py --rank 0 --mode ep --iters 5 >> gpurun_out/p8_layout_r02_v2.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:grouped_gemm \
  -s 6 -c 2 -o gpurun_out/prof_p8gemm_r02_v2 python tools/p8_layout_gemm.py --rank 1 --iters 5 > gpurun_out/ncu_p8_r02_v2.log 2>&1
tail -30 gpurun_out/pytest_r02_v2.log; cat gpurun_out/p8_layout_r02_v2.jsonl; tail -c 600 gpurun_out/bench_r02_v2_p2share.err; head -c 600 gpurun_out/bench_r02_v2_p2share.json
