#!/bin/bash
# Same-box A/B of the weight-gradient GEMM across library builds (tools/ab_variant.sh outputs):
# P=8 critical-rank layout (dW13, dW_down) and the P=1 layout, twice each, alternating builds.
# usage: tools/wgrad_ab.sh lib1 lib2 ...   (outputs must agree bitwise: same sha1 per shape)
for rep in $(seq 1 ${REPS:-2}); do
  for lib in "$@"; do
    for shape in "p8 5760 2880" "p8 2880 2880" "both 5760 2880"; do
      echo "$lib $(LLEP_LIB=$lib timeout 120 python tools/wgrad_bench.py $shape 2>&1 | tail -1)"
    done
  done
done
