timeout 900 python -m pytest tests/test_gpu_backward.py -x -q > gpurun_out/pytest_bwd_v5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bwd_v5.log
python tools/fwd_ab.py LLEP_BWD_UNFUSED 1 0 --train --reps 2 --secs 4 > gpurun_out/bwd_ab_fuse.jsonl 2>&1
python tools/fwd_ab.py LLEP_BWD_UNFUSED 1 0 --train --reps 2 --secs 4 --config q3 >> gpurun_out/bwd_ab_fuse.jsonl 2>&1
tail -3 gpurun_out/pytest_bwd_v5.log; cat gpurun_out/bwd_ab_fuse.jsonl
