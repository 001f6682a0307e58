#!/bin/bash
# fused combine (P = 1): correctness, then in-situ A/B against the separate combine kernel
mkdir -p gpurun_out
python -m pytest tests/test_gpu_layer.py -x -q -k "fused_combine or p1_full or empty_and_small or g120_p1 or q3_p1 or local_gather or multicast" > gpurun_out/fused_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/fused_pytest.log
python -m pytest tests/test_gpu_graph.py tests/test_gpu_kernels.py -x -q >> gpurun_out/fused_pytest.log 2>&1
echo "pytest2 exit $?" >> gpurun_out/fused_pytest.log
for cfg in g120 q3 dsv3; do
  timeout 300 python tools/fwd_ab.py LLEP_FUSED_COMBINE 0 1 --config $cfg --secs 3 >> gpurun_out/fused_ab.jsonl 2>&1
done
for hot in 0; do
  timeout 300 python tools/fwd_ab.py LLEP_FUSED_COMBINE 0 1 --config g120 --hot $hot --secs 3 >> gpurun_out/fused_ab.jsonl 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/fused_bench.json 2> gpurun_out/fused_bench.err
tail -3 gpurun_out/fused_pytest.log; cat gpurun_out/fused_ab.jsonl; cat gpurun_out/fused_bench.json
