export LLEP_BENCH_SHARE_GPU=1 LLEP_BENCH_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus 2 --steps 3 --warmup 3 --config g20 > gpurun_out/bench_p2_shared.json 2> gpurun_out/bench_p2_shared.err; echo "rc=$?" >> gpurun_out/bench_p2_shared.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29912 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_ref_p2.json 2> gpurun_out/bench_ref_p2.err; echo "rc=$?" >> gpurun_out/bench_ref_p2.err
tail -2 gpurun_out/bench_p2_shared.err; cut -c1-400 gpurun_out/bench_p2_shared.json; tail -1 gpurun_out/bench_ref_p2.err; cut -c1-200 gpurun_out/bench_ref_p2.json
