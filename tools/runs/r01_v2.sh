python tools/layout_ab.py g120p1 dense > gpurun_out/layout_ab.jsonl 2>&1
python tools/layout_ab.py hot cold >> gpurun_out/layout_ab.jsonl 2>&1
python tools/layout_ab.py g120p8 uniform16 >> gpurun_out/layout_ab.jsonl 2>&1
python tools/wgrad_bench.py small 5760 2880 > gpurun_out/wgrad_v2.txt 2>&1
python tools/wgrad_bench.py hot 5760 2880 >> gpurun_out/wgrad_v2.txt 2>&1
python tools/wgrad_bench.py both 5760 2880 >> gpurun_out/wgrad_v2.txt 2>&1
ncu --set full --clock-control none --kernel-name-base mangled -k regex:gemm_bwd_pair -s 3 -c 1 -o gpurun_out/prof_wgrad_small python tools/wgrad_bench.py small 5760 2880 > /dev/null 2>&1
cat gpurun_out/layout_ab.jsonl gpurun_out/wgrad_v2.txt
