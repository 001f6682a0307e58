#!/bin/bash
# A/B of grouped-GEMM variants at fixed (base) clocks: duration + tensor-pipe activity per launch.
# usage: tools/ab_ncu.sh <layout> [variants] [iters]
L=${1:-g120p1}; V=${2:-cta1,cta2}; IT=${3:-1}
ncu --clock-control base --metrics gpu__time_duration.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum \
    -k regex:grouped_gemm --csv python tools/gemm_bench.py --layout $L --iters $IT --variants $V $GB_ARGS 2>/dev/null \
  | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d={}
for r in rows[1:]:
    d.setdefault((int(r[ii]),r[ki][:48]),{})[r[mi]]=r[vi]
for k,v in sorted(d.items()):
    print(k[0], k[1], 'ns', v.get('gpu__time_duration.sum'), 'tensor%', v.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'), 'dram', v.get('dram__bytes_read.sum'))
"
