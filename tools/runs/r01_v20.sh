for c in g20 fhead q3 dsv3 kimi; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_f3_$c.json 2> gpurun_out/bench_f3_$c.err; done
for c in g20 fhead q3 dsv3 kimi; do python -c "
import json;d=json.load(open('gpurun_out/bench_f3_$c.json'))
r=d['roofline']; b=d.get('backward',{})
print('$c', round(d['value']/1e6,2), round(d['ms_per_step'],2), round(r['achieved']), round(r['gemm2_tflops']), round(b.get('ms_per_step',0),1), round(b.get('tflops',0)), round(b.get('train_step',{}).get('ms_per_step',0),1), round(d['peak_gb_per_gpu'],1), round(d['router']['ms_per_call']*1e3,1), d['clocks']['sm_mhz'])
"; done
