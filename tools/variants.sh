cd $GRAFT_REPO_ROOT
for v in "$@"; do
  cp paper_2309_09025_b200/libfdsnn_b200_$v.so paper_2309_09025_b200/libfdsnn_b200.so
  echo "== $v"; python tools/perf_probe.py 4096 16384 2>&1 | tail -2
done
