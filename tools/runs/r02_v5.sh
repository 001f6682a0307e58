# round 2, pass 5: sliding-window L2 prefetch of the swapped (cold-expert) tiles' weights, A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02_v5.log 2>&1
for pf in 1 2 4 8; do timeout 300 python tools/fwd_ab.py LLEP_SWAP_PF 0 $pf --config g120 --hot 95 --secs 4; done > gpurun_out/ab_swap_pf_g120.jsonl 2>&1
for pf in 2 4; do timeout 300 python tools/fwd_ab.py LLEP_SWAP_PF 0 $pf --config dsv3 --hot 95 --secs 4; done > gpurun_out/ab_swap_pf_dsv3.jsonl 2>&1
for pf in 2 4; do timeout 300 python tools/fwd_ab.py LLEP_SWAP_PF 0 $pf --config q3 --hot 95 --secs 4; done > gpurun_out/ab_swap_pf_q3.jsonl 2>&1
cat gpurun_out/ab_swap_pf_*.jsonl
