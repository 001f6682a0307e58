python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_v26.log 2>&1; tail -1 gpurun_out/smoke_v26.log
timeout 1800 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest_r02_v26.log 2>&1; echo rc=$? >> gpurun_out/pytest_r02_v26.log
tail -4 gpurun_out/pytest_r02_v26.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02_v26.json 2> gpurun_out/bench_r02_v26.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_r02_v26.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'], d['graph'].get('ms_per_step'), d['e2e']['value'])"
