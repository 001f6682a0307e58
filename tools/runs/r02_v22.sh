python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in 1 2 3; do timeout 300 python tools/fwd_ab.py LLEP_L2_HOT 0 $v --config g120 --hot 95 --secs 4; done > gpurun_out/ab_l2hot_g120.jsonl 2>&1
for v in 1 3; do timeout 300 python tools/fwd_ab.py LLEP_L2_HOT 0 $v --config q3 --hot 95 --secs 3; done > gpurun_out/ab_l2hot_q3.jsonl 2>&1
for v in 1; do timeout 300 python tools/fwd_ab.py LLEP_L2_HOT 0 $v --config g120 --hot 0 --secs 3; done > gpurun_out/ab_l2hot_bal.jsonl 2>&1
cat gpurun_out/ab_l2hot_*.jsonl
