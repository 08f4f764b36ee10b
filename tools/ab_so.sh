# A/B the in-tree library against tools/ab_A.so (a build of other sources):
#   bash tools/ab_so.sh [probe sizes...]   (PROBE_PARAMS=c4 for C4)
cd $GRAFT_REPO_ROOT
L=paper_2309_09025_b200
cp $L/libfdsnn_b200.so /tmp/B.so
for v in A B A B; do
  if [ $v = A ]; then cp tools/ab_A.so $L/libfdsnn_b200.so; else cp /tmp/B.so $L/libfdsnn_b200.so; fi
  echo "== $v"; timeout 300 python tools/perf_probe.py "$@" 2>&1 | grep "^B="
done
cp /tmp/B.so $L/libfdsnn_b200.so
