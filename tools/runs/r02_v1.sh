# round 2, first GPU pass: full GPU suite (timed per test) + bench line
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_r02_v1.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/pytest_r02_v1.log 2>&1; echo rc=$? >> gpurun_out/pytest_r02_v1.log
timeout 600 python bench.py > gpurun_out/bench_r02_v1.json 2> gpurun_out/bench_r02_v1.err
tail -45 gpurun_out/pytest_r02_v1.log; tail -c 1500 gpurun_out/bench_r02_v1.err
