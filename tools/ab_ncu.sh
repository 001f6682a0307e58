#!/bin/bash
# A/B of grouped-GEMM variants at fixed (base) clocks: duration + tensor-pipe activity per launch.
# usage: tools/ab_ncu.sh <layout> [iters]
L=${1:-g120p1}; IT=${2:-2}
ncu --clock-control base --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum \
    -k regex:grouped_gemm --csv python tools/gemm_bench.py --layout $L --iters $IT 2>/dev/null \
  | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
from collections import OrderedDict
d=OrderedDict()
for r in rows[1:]:
    d.setdefault((int(r[ii]),r[ki][:40]),{})[r[mi]]=r[vi]
per=int('$IT')+3
items=list(d.items())
variants=['interleave','group_order']*2
for n,(k,v) in enumerate(items):
    blk=n//per; var=variants[(blk//2)%4] if False else None
    print(k[0], k[1], v.get('gpu__time_duration.sum'), 'tensor%', v.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'), 'dram', v.get('dram__bytes_read.sum'))
"
