#!/bin/bash
# Weight-gradient GEMM A/B at base clocks (ncu --clock-control base: power-cap noise removed), per build:
# kernel time and tensor-pipe activity of the pair wgrad kernel and its split-K reduce (sum per call) on the P=8 critical-rank layout and P=1.
# usage: tools/wgrad_ab_ncu.sh lib1 lib2 ...
for lib in "$@"; do
  for shape in "p8 5760 2880" "p8 2880 2880" "both 5760 2880"; do
    LLEP_LIB=$lib ncu --clock-control base --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
        -k regex:"gemm_bwd_pair|split_reduce" -s 4 -c 4 --csv python tools/wgrad_bench.py $shape 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
rows=rows[next(i for i,r in enumerate(rows) if r[0]=='ID'):]
h=rows[0]; mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d={}
for r in rows[1:]:
    d.setdefault(int(r[ii]),{})[r[mi]]=r[vi]
print('$lib'.split('/')[-2], '$shape', ' | '.join('%s us, tensor %s%%' % (float(v['gpu__time_duration.sum'].replace(',',''))/1e3, v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']) for k,v in sorted(d.items())), '| sum/2 %.1f us' % (sum(float(v['gpu__time_duration.sum'].replace(',','')) for v in d.values())/2e3))
"
  done
done
