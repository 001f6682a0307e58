set -x
python tools/mem_sweep.py --config g120 --world 8 --scenarios 95:1,95:4,95:16,50:1,30:1,0:0 > gpurun_out/mem_g120_p8.jsonl 2> gpurun_out/mem_g120_p8.err
python tools/mem_sweep.py --config g120 --world 4 --scenarios 95:1,0:0 --port 29760 > gpurun_out/mem_g120_p4.jsonl 2> gpurun_out/mem_g120_p4.err
python tools/mem_sweep.py --config g120 --world 2 --scenarios 95:1,0:0 --port 29770 > gpurun_out/mem_g120_p2.jsonl 2> gpurun_out/mem_g120_p2.err
python tools/mem_sweep.py --config g20 --world 8 --scenarios 95:1 --port 29780 > gpurun_out/mem_g20_p8.jsonl 2> gpurun_out/mem_g20_p8.err
python tools/mem_sweep.py --config q3 --world 8 --scenarios 95:1,0:0 --port 29790 > gpurun_out/mem_q3_p8.jsonl 2> gpurun_out/mem_q3_p8.err
python tools/emulate_p8.py --world 4 --scenarios 95:1,80:1,50:1,30:1,95:4,95:16,0:0 > gpurun_out/emu_g120_p4.jsonl 2>&1
python tools/emulate_p8.py --world 2 --scenarios 95:1,80:1,50:1,30:1,95:4,95:16,0:0 > gpurun_out/emu_g120_p2.jsonl 2>&1
python tools/emulate_p8.py --config g20 --world 8 --scenarios 95:1,50:1,0:0 > gpurun_out/emu_g20_p8.jsonl 2>&1
python tools/emulate_p8.py --config q3 --world 8 --scenarios 95:1,50:1,0:0 > gpurun_out/emu_q3_p8.jsonl 2>&1
