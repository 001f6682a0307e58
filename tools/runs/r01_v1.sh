timeout 900 python -m pytest tests/test_gpu_backward.py -x -q > gpurun_out/pytest_bwd_v1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bwd_v1.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v1.json 2> gpurun_out/bench_v1.err
python tools/emulate_p8.py --world 2 --scenarios 95:4,0:0,95:1 --reps 4 > gpurun_out/emu_recheck.jsonl 2>&1
python tools/emulate_p8.py --config g20 --world 8 --scenarios 0:0,95:1 --reps 4 >> gpurun_out/emu_recheck.jsonl 2>&1
tail -2 gpurun_out/pytest_bwd_v1.log
