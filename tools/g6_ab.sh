# A/B: 12-warp CTAs (6 rotations, 168 registers, 3-stage ring) vs 8-warp (dev aid)
cd $GRAFT_REPO_ROOT
FDSNN_G6=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for d in 1 0; do echo "G6=$d"; FDSNN_G6=$d timeout 300 python tools/perf_probe.py 2664 8880 2>&1 | tail -2; done
FDSNN_G6=1 ncu --set full --clock-control none --import-source on -k regex:pbs_blind -s 1 -c 1 -o gpurun_out/g6_br python tools/prof_target.py 2664 > gpurun_out/g6_ncu.log 2>&1; echo "ncu rc=$?"
