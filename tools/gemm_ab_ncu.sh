#!/bin/bash
# Forward pair GEMMs at base clocks (ncu --clock-control base), standalone entry (tools/gemm_bench.py,
# g120p1 layout) per library build: time and tensor-pipe activity of GEMM1 / GEMM2 launches.
# usage: tools/gemm_ab_ncu.sh lib1 lib2 ...
for lib in "$@"; do
  LLEP_LIB=$lib ncu --clock-control base --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
      -k regex:grouped_gemm_2cta -s 6 -c 4 --csv python tools/gemm_bench.py --layout ${LAYOUT:-g120p1} --variants cta2 --iters 3 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
rows=rows[next(i for i,r in enumerate(rows) if r[0]=='ID'):]
h=rows[0]; mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID'); ki=h.index('Kernel Name')
d={}
for r in rows[1:]:
    d.setdefault((int(r[ii]), r[ki].split('(')[0][-40:]),{})[r[mi]]=r[vi]
print('$lib', ' | '.join('%s %s us tensor %s%%' % (k[1], float(v['gpu__time_duration.sum'].replace(',',''))/1e3, v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']) for k,v in sorted(d.items())))
"
done
