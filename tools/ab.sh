# A/B of blind-rotation kernels: warp-per-accumulator vs group
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x -k "desk or ragged or determin or margin or empty" 2>&1 | tail -2
for k in warp group; do echo "== $k"; FDSNN_BR_KERNEL=$k python tools/perf_probe.py 4096 16384 2>&1 | tail -2; done
