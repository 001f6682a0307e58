python tools/fwd_ab.py LLEP_BWD_UNFUSED 1 0 --train --reps 2 --secs 4 > gpurun_out/bwd_ab_fuse.jsonl 2>&1
python tools/fwd_ab.py LLEP_BWD_UNFUSED 1 0 --train --reps 2 --secs 4 --config q3 >> gpurun_out/bwd_ab_fuse.jsonl 2>&1
python tools/fwd_ab.py LLEP_BWD_UNFUSED 0 1 --train --reps 2 --secs 4 >> gpurun_out/bwd_ab_fuse.jsonl 2>&1
cat gpurun_out/bwd_ab_fuse.jsonl
