# ncu --set full of one DESK blind-rotation launch (dev aid): bash tools/prof_br.sh <tag>
cd $GRAFT_REPO_ROOT
python tools/prof_target.py 2368 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:pbs_blind -s 1 -c 1 -o gpurun_out/$1_br python tools/prof_target.py 2368 > gpurun_out/$1_ncu.log 2>&1; echo "ncu rc=$?"
