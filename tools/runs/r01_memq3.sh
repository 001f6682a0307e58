python tools/mem_sweep.py --config q3 --world 8 --scenarios 95:1,0:0 --port 29790 --modes llep > gpurun_out/mem_q3_p8.jsonl 2> gpurun_out/mem_q3_p8.err
