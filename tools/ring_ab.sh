# A/B of the key-ring depth (dev aid): FDSNN_RING_S = 3, 4 (default), 5
cd $GRAFT_REPO_ROOT
B=paper_2309_09025_b200
cp $B/libfdsnn_b200.so /tmp/s4.so
for S in 3 5; do
  (cd $B/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
      -diag-suppress 177,1886 -DFDSNN_RING_S=$S -o /tmp/s$S.so capi.cu)
done
for S in 4 3 5 4; do cp /tmp/s$S.so $B/libfdsnn_b200.so; echo "S=$S"; timeout 300 python tools/perf_probe.py 2048 8192 2>&1 | tail -2; done
cp /tmp/s4.so $B/libfdsnn_b200.so
