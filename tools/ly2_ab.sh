# A/B of the layout-2 blind rotation vs the Stockham PAIR variant (dev aid)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q 2>&1 | tail -2
timeout 300 python tools/perf_probe.py 2048 8192 2>&1 | tail -2
cp paper_2309_09025_b200/libfdsnn_b200.so /tmp/ly2.so
cd paper_2309_09025_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -diag-suppress 177,1886 -DFDSNN_LY2=0 -o ../libfdsnn_b200.so capi.cu && cd ../..
timeout 300 python tools/perf_probe.py 2048 8192 2>&1 | tail -2
cp /tmp/ly2.so paper_2309_09025_b200/libfdsnn_b200.so
