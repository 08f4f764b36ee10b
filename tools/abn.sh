# A/B/C... of compile-time variants of the library (dev aid):
#   bash tools/abn.sh "-DFOO=1" "-DBAR=2" ...   (PROBE="2048 8192" to change sizes)
# Variant 0 is the in-tree build.  Every variant first runs the parity/golden
# GPU tests, then the perf probe runs round-robin over the variants twice.
cd $GRAFT_REPO_ROOT
SIZES=${PROBE:-"8192"}
L=paper_2309_09025_b200
cp $L/libfdsnn_b200.so /tmp/V0.so
i=1
for F in "$@"; do
  (cd $L/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
      -diag-suppress 177,1886 $F -o /tmp/V$i.so capi.cu) &
  i=$((i+1))
done
wait
NV=$i
for ((v=1; v<NV; v++)); do
  cp /tmp/V$v.so $L/libfdsnn_b200.so
  echo "== tests V$v: $(timeout 300 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_golden.py} -x -q 2>&1 | tail -1)"
done
for rep in 1 2; do
  for ((v=0; v<NV; v++)); do
    cp /tmp/V$v.so $L/libfdsnn_b200.so
    echo "== V$v $(timeout 150 python tools/perf_probe.py $SIZES 2>&1 | grep '^B=')"
  done
done
cp /tmp/V0.so $L/libfdsnn_b200.so
