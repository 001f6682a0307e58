python tools/layout_ab.py cold cold128 > gpurun_out/layout_ab3.jsonl 2>&1
python tools/layout_ab.py cold256 cold64g >> gpurun_out/layout_ab3.jsonl 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:grouped_gemm_2cta -s 6 -c 2 -o gpurun_out/prof_cold python tools/layout_ab.py cold dense > /dev/null 2>&1
cat gpurun_out/layout_ab3.jsonl
