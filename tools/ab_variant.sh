#!/bin/bash
# Build an A/B variant of libllep.so with extra -D flags for gemm.cu only (the other objects are the
# default build's): tools/ab_variant.sh NAME "-DX=1 -DY=2"  ->  paper_2601_17111_b200/_ab/NAME/libllep.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
PKG=$ROOT/paper_2601_17111_b200
python -m paper_2601_17111_b200.build > /dev/null
OUT=$PKG/_ab/$1
mkdir -p $OUT
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
  --expt-relaxed-constexpr -I $ROOT/include -I $PKG/csrc $2 -c $PKG/csrc/gemm.cu -o $OUT/gemm.cu.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libllep.so $PKG/_build/api.cu.o \
  $PKG/_build/plan.cu.o $PKG/_build/route.cu.o $OUT/gemm.cu.o $PKG/_build/router.cu.o -cudart static
echo $OUT/libllep.so
