#!/bin/bash
# A/B of the backward GEMMs of two library builds at base clocks (ncu), G120 P=1 bench workload.
# usage: tools/ab_bwd.sh <libA> <libB>
for lib in $1 $2 $1 $2; do
  echo "== $lib"
  LLEP_LIB=$lib ncu --clock-control base --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
      -k regex:"gemm_bwd_pair|grouped_gemm_2cta_kernel<240, 2" -c 10 --csv \
      python bench.py --no-e2e --no-cpu-baseline --steps 1 --warmup 3 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
rows=rows[next(i for i,r in enumerate(rows) if r[0]=='ID'):]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d={}
for r in rows[1:]:
    d.setdefault((int(r[ii]),r[ki][:40]),{})[r[mi]]=r[vi]
for k,v in sorted(d.items()):
    print(k[0], k[1], 'ns', v.get('gpu__time_duration.sum'), 'tensor%', v.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'))
"
done
