# round 2, pass 7: hot-group GEMM efficiency vs operand-ring size / BN (sizing a dual hot+cold pipeline)
for v in default bn192 bn192_k1_112 bn192_k2_112 bn240_k1_112; do
  if [ $v = default ]; then unset LLEP_LIB; else export LLEP_LIB=paper_2601_17111_b200/_ab/$v/libllep.so; fi
  echo "== $v"
  timeout 300 python tools/gemm_bench.py --layout hot --variants cta2 --iters 20 | tail -2
  timeout 300 python tools/gemm_bench.py --layout hot --D 7168 --H 2048 --variants cta2 --iters 10 | tail -2
done > gpurun_out/ring_ab.txt 2>&1
unset LLEP_LIB
cat gpurun_out/ring_ab.txt
