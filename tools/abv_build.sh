#!/bin/bash
# Build library variants for tools/abv.sh: bash tools/abv_build.sh "-DFOO=1" "-DBAR=2" ...
cd "$(dirname "$0")/.."
mkdir -p tools/ab && rm -f tools/ab/V*.so
i=1
for F in "$@"; do
  (cd paper_2309_09025_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
      -Xcompiler -fPIC -diag-suppress 177,1886 $F -o ../../tools/ab/V$i.so capi.cu && echo "V$i: $F") &
  i=$((i+1))
done
wait
