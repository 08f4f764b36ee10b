#!/bin/bash
# Development cycle on the GPU box: parity tests, timing probe, optional ncu capture.
# usage: bash tools/gpu_cycle.sh <tag> [ncu]
TAG=${1:-dev}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
python tools/perf_probe.py 4096 16384 > gpurun_out/${TAG}_perf.log 2>&1; cat gpurun_out/${TAG}_perf.log
if [ "$2" == "ncu" ]; then
  python tools/prof_target.py 592 > gpurun_out/${TAG}_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:pbs_blind -s 1 -c 1 -o gpurun_out/${TAG}_br python tools/prof_target.py 592 > gpurun_out/${TAG}_ncu.log 2>&1
  tail -2 gpurun_out/${TAG}_ncu.log
fi
