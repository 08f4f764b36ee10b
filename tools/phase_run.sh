# build the phase-profiling variant into /tmp and run the probe with it
cd $GRAFT_REPO_ROOT
L=paper_2309_09025_b200
cp $L/libfdsnn_b200.so /tmp/A.so
(cd $L/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
    -diag-suppress 177,1886,128 -DFDSNN_PHASE_PROF $EXTRA -o /tmp/P.so capi.cu) || exit 1
cp /tmp/P.so $L/libfdsnn_b200.so
for B in "$@"; do echo "== B=$B"; python tools/phase_probe.py $B; done
cp /tmp/A.so $L/libfdsnn_b200.so
