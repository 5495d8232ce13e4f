#!/bin/bash
# build libgradsync_b200 variants with different pass-1 tuning macros into
# tools/variants/ (only gs_lars.cu is recompiled; the rest comes from the
# main build's objects)
set -e
cd "$(dirname "$0")/.."
python paper_1807_11205_b200/_build.py > /dev/null
mkdir -p tools/variants
rm -f tools/variants/*.so
for v in "$@"; do
  r=${v%x*}; m=${v#*x}
  out=tools/variants/lib_r${r}_m${m}.so
  o=/tmp/var_${r}_${m}_gs_lars.o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC \
    -I include -DGS_P1_ROUNDS=$r -DGS_P1_MINB=$m -c paper_1807_11205_b200/csrc/gs_lars.cu -o $o &
  wait
  objs=$(ls paper_1807_11205_b200/_lib/obj/*.o | grep -v gs_lars.o)
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o $out $objs $o
  echo built $out
done
