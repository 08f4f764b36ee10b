#!/bin/bash
# Static SASS opcode counts of the PAIR blind-rotation kernel (dev aid, no GPU):
#   tools/sass_static.sh [-DFOO=1 ...]
D=$(mktemp -d)
cat > $D/k.cu <<'EOT'
#include "pbs.cuh"
template __global__ void fdsnn::pbs_blind_rotate_kernel<512, 4, false, false, true>(fdsnn::PbsArgs);
EOT
R=$(cd "$(dirname "$0")/.." && pwd)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I $R/paper_2309_09025_b200/csrc -cubin \
    -diag-suppress 177,1886 -Xptxas -v "$@" -o $D/k.cubin $D/k.cu 2>&1 | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores"
cuobjdump -sass $D/k.cubin | grep -oP '^\s+/\*[0-9a-f]+\*/\s+\K(@!?U?P[0-9T] )?[A-Z0-9_.]+' | sed 's/^@[!A-Z0-9]* //' |
    awk '{split($1,a,"."); o=a[1]; if (o=="IMAD" && $1 ~ /MOV/) o="IMAD.MOV"; c[o]++; n++} END {for (k in c) printf "%-10s %5d\n", k, c[k]; printf "%-10s %5d\n", "TOTAL", n}' |
    sort -k2 -nr | head -${TOPN:-16} | tr '\n' ' '; echo
rm -rf $D
