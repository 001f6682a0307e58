# row f3 ablations with the round-2 code and the chunk-aligned link model
timeout 3000 python tools/ablate.py --reps 2 > gpurun_out/ablations_r02.jsonl 2> gpurun_out/ablations_r02.err
wc -l gpurun_out/ablations_r02.jsonl; tail -3 gpurun_out/ablations_r02.err
