# Timing ablation (dev aid, results invalid): refill 1/2 or 1/16 of each key chunk
cd $GRAFT_REPO_ROOT
B=paper_2309_09025_b200
cp $B/libfdsnn_b200.so /tmp/base.so
for v in base tools/abl_k2 tools/abl_k16 base; do
  if [ $v = base ]; then cp /tmp/base.so $B/libfdsnn_b200.so; else cp $v.so $B/libfdsnn_b200.so; fi
  echo "$v"; timeout 300 python tools/perf_probe.py 2048 8192 2>&1 | tail -2
done
cp /tmp/base.so $B/libfdsnn_b200.so
