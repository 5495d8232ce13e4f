#!/bin/bash
# build libgradsync_b200 variants with different pass-1 tuning macros into tools/variants/
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/variants
for v in "$@"; do
  r=${v%x*}; m=${v#*x}
  out=tools/variants/lib_r${r}_m${m}.so
  objs=""
  for f in paper_1807_11205_b200/csrc/*.cu; do
    o=/tmp/var_${r}_${m}_$(basename $f .cu).o
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC \
      -I include -DGS_P1_ROUNDS=$r -DGS_P1_MINB=$m -c $f -o $o
    objs="$objs $o"
  done
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o $out $objs
  echo built $out
done
