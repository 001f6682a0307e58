# round 2, pass 12: refresh of the secondary measurements with the round-2 code
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02_v12.log 2>&1
( timeout 300 python tools/wgrad_bench.py p8 2880 2880; timeout 300 python tools/wgrad_bench.py p8 5760 2880 ) > gpurun_out/wgrad_p8.txt 2>&1
timeout 900 python tools/emulate_p8.py > gpurun_out/emulate_p8_r02.jsonl 2> gpurun_out/emulate_p8_r02.err
for c in g20 fhead q3 dsv3 kimi; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-distinct > gpurun_out/f3_$c.json 2> gpurun_out/f3_$c.err; done
cat gpurun_out/wgrad_p8.txt; cat gpurun_out/emulate_p8_r02.jsonl | cut -c1-400
for c in g20 fhead q3 dsv3 kimi; do python -c "
import json,sys; d=json.loads(open('gpurun_out/f3_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']), round(d['roofline']['gemm2_tflops']), d['backward']['ms_per_step'] if 'backward' in d else None, d['peak_gb_per_gpu'], d['clocks']['sm_mhz'])"; done
