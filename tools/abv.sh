#!/bin/bash
# Time prebuilt library variants (dev aid): tools/ab/V*.so are built in the
# build container (tools/abv_build.sh) and shipped with the snapshot; V0 is
# the in-tree build.  usage: bash tools/abv.sh [probe sizes]   (TESTS=1: parity tests first)
cd $GRAFT_REPO_ROOT
SIZES=${@:-8192}
L=paper_2309_09025_b200
cp $L/libfdsnn_b200.so /tmp/V0.so
VS="/tmp/V0.so $(ls tools/ab/V*.so 2>/dev/null)"
if [ -n "$TESTS" ]; then
  for v in $VS; do
    cp $v $L/libfdsnn_b200.so
    echo "== tests $(basename $v): $(timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q 2>&1 | tail -1)"
  done
fi
for rep in 1 2; do
  for v in $VS; do
    cp $v $L/libfdsnn_b200.so
    echo "== $(basename $v) $(timeout 150 python tools/perf_probe.py $SIZES 2>&1 | grep '^B=')"
  done
done
cp /tmp/V0.so $L/libfdsnn_b200.so
