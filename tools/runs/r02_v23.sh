for w in 2 4; do timeout 900 python tools/emulate_p8.py --world $w; done > gpurun_out/emulate_sweep_r02.jsonl 2> gpurun_out/emulate_sweep_r02.err
wc -l gpurun_out/emulate_sweep_r02.jsonl
