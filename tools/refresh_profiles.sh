#!/bin/bash
# Round-end evidence on one GPU: parity tests, the default bench line, the ncu
# launch list of the bench command and one `--set full` capture of the blind
# rotation kernel inside the bench (each ncu pass only after the same command
# exited 0 without ncu).  usage: bash tools/refresh_profiles.sh <tag>
TAG=${1:-final}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/${TAG}_tests.log
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"; cat $O/${TAG}_bench.json
python tools/perf_configs.py > $O/${TAG}_configs.log 2>&1; echo "configs rc=$?"; tail -12 $O/${TAG}_configs.log
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
if $CMD > $O/${TAG}_plain.json 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launch.log 2>&1; echo "launch list rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:pbs_br16 -s 3 -c 1 \
      -o $O/${TAG}_bench_br $CMD > $O/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
  tail -2 $O/${TAG}_ncu_full.log
fi
