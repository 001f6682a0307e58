#!/bin/bash
# Backward row GEMMs (kind 0) at base clocks per build: time and tensor-pipe activity, P=8 layout and P=1.
# usage: tools/bwd_rows_ncu.sh lib1 lib2 ...
for lib in "$@"; do
  IFS=, read -ra SH <<< "${SHAPES:-p8 2880 2880,p8 5760 2880,both 5760 2880}"
  for shape in "${SH[@]}"; do
    LLEP_LIB=$lib ncu --clock-control base --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum \
        -k regex:gemm_bwd_pair -s 2 -c 2 --csv python tools/bwd_rows_bench.py $shape 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
rows=rows[next(i for i,r in enumerate(rows) if r[0]=='ID'):]
h=rows[0]; mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d={}
for r in rows[1:]:
    d.setdefault(int(r[ii]),{})[r[mi]]=r[vi]
print('$lib'.split('/')[-2], '${TAG:-}', '$shape', ' | '.join('%s us, tensor %s%%, dram %s, xbar %s' % (float(v['gpu__time_duration.sum'].replace(',',''))/1e3, v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'], v['dram__bytes_read.sum'], v['l1tex__m_xbar2l1tex_read_bytes.sum']) for k,v in sorted(d.items())))
"
  done
done
