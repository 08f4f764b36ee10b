# ncu capture of the C4 (N=2048) blind rotation (dev aid)
cd $GRAFT_REPO_ROOT
O=gpurun_out
PROBE_PARAMS=c4 timeout 300 python tools/perf_probe.py 1184 2>&1 | tail -1
PROBE_PARAMS=c4 python tools/prof_target.py 1184 > /dev/null 2>&1 || exit 1
PROBE_PARAMS=c4 ncu --set full --clock-control none --import-source on -k regex:pbs_blind -s 1 -c 1 -o $O/c4c_br python tools/prof_target.py 1184 > $O/c4c_ncu.log 2>&1; echo "ncu rc=$?"
