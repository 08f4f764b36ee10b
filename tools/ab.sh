# A/B a compile-time variant of the library (dev aid):
#   bash tools/ab.sh "-DFOO=0" [probe sizes...]
# Runs the parity/golden GPU tests on the in-tree (default) build, then the
# perf probe alternately on the default build (A) and the variant (B).
cd $GRAFT_REPO_ROOT
FLAGS=$1; shift
SIZES=${@:-2048 8192}
L=paper_2309_09025_b200
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q 2>&1 | tail -1
cp $L/libfdsnn_b200.so /tmp/A.so
(cd $L/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
    -diag-suppress 177,1886 $FLAGS -o /tmp/B.so capi.cu) || exit 1
for v in A B A B; do
  cp /tmp/$v.so $L/libfdsnn_b200.so; echo "== $v"
  timeout 300 python tools/perf_probe.py $SIZES 2>&1 | grep "^B="
done
cp /tmp/A.so $L/libfdsnn_b200.so
