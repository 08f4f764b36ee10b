# A/B of a compile-time variant on the C4 (N=2048) blind rotation (dev aid): bash tools/ab_c4.sh "-DFOO=0"
cd $GRAFT_REPO_ROOT
L=paper_2309_09025_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q 2>&1 | tail -1
cp $L/libfdsnn_b200.so /tmp/A.so
(cd $L/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
    -diag-suppress 177,1886 $1 -o /tmp/B.so capi.cu) || exit 1
for v in A B A B; do
  cp /tmp/$v.so $L/libfdsnn_b200.so; echo "== $v"
  PROBE_PARAMS=c4 timeout 300 python tools/perf_probe.py 1184 2368 2>&1 | grep "^B="
done
cp /tmp/A.so $L/libfdsnn_b200.so
