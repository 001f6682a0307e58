#!/bin/bash
# Build an A/B variant of libllep.so with extra -D flags for ALL sources (tools/ab_variant.sh does gemm.cu
# only): tools/ab_variant_all.sh NAME "-DX=1"  ->  paper_2601_17111_b200/_ab/NAME/libllep.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
PKG=$ROOT/paper_2601_17111_b200
OUT=$PKG/_ab/$1
mkdir -p $OUT
for s in api plan route gemm router; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
    --expt-relaxed-constexpr -I $ROOT/include -I $PKG/csrc $2 -c $PKG/csrc/$s.cu -o $OUT/$s.cu.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libllep.so $OUT/api.cu.o \
  $OUT/plan.cu.o $OUT/route.cu.o $OUT/gemm.cu.o $OUT/router.cu.o -cudart static
echo $OUT/libllep.so
