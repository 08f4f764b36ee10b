cd $GRAFT_REPO_ROOT
for v in "$@"; do
  cp paper_2309_09025_b200/libfdsnn_b200_$v.so paper_2309_09025_b200/libfdsnn_b200.so
  echo "== $v"; FDSNN_BR_KERNEL=group python tools/perf_probe.py 16384 2>&1 | tail -1
done
