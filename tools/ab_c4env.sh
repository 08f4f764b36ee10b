# A/B of an environment switch on the C4 blind rotation (dev aid): bash tools/ab_c4env.sh VAR
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_golden.py -x -q 2>&1 | tail -1
for v in 1 0 1 0; do echo "== $1=$v"; env $1=$v PROBE_PARAMS=c4 timeout 300 python tools/perf_probe.py 1184 2368 2>&1 | grep "^B="; done
