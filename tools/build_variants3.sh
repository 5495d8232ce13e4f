#!/bin/bash
# pass-1 variants: ROUNDSxMINBxWIDEN (GS_P1_ROUNDS, GS_P1_MINB, GS_P1_WIDEN)
# -> tools/variants/lib_<spec>.so (only gs_lars.cu recompiled)
set -e
cd "$(dirname "$0")/.."
python -c "from paper_1807_11205_b200 import _build; _build.build()" > /dev/null
mkdir -p tools/variants
rm -f tools/variants/*.so
objs=$(ls paper_1807_11205_b200/_lib/obj/*.o | grep -v gs_lars.o)
for v in "$@"; do
  IFS=x read r m w <<< "$v"
  (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC \
    -I include -DGS_P1_ROUNDS=$r -DGS_P1_MINB=$m -DGS_P1_WIDEN=$w -c paper_1807_11205_b200/csrc/gs_lars.cu \
    -o /tmp/var_$v.o && nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static \
    -o tools/variants/lib_$v.so $objs /tmp/var_$v.o && echo built $v) &
done
wait
