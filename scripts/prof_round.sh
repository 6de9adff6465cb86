#!/bin/bash
# The round's profiling pass (one B200, under gpurun): plain bench run, the launch list of the
# same command, and ncu --set full captures of every kernel the bench line reports.
# Usage: bash scripts/prof_round.sh <tag>   -> gpurun_out/prof_<tag>/
set -u
TAG=${1:-r2}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > $OUT/plain.log 2>&1 || { echo "plain run failed"; tail $OUT/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
FULL="ncu --set full --clock-control none --import-source on"
$FULL -k regex:rollout_mlp -c 1 -o $OUT/mlp python bench.py --steps 1 --warmup 0 --no-secondary --no-cpu-baseline --T 1000 > $OUT/ncu_mlp.log 2>&1
$FULL -k regex:step_kernel -s 10 -c 1 -o $OUT/step python scripts/run_step.py > $OUT/ncu_step.log 2>&1
$FULL -k regex:rollout_open -c 1 -o $OUT/open_dyn python scripts/run_open.py dyn > $OUT/ncu_open_dyn.log 2>&1
$FULL -k regex:rollout_open -c 1 -o $OUT/open_c5 python scripts/run_open.py c5 > $OUT/ncu_open_c5.log 2>&1
$FULL -k regex:track_mlp -c 1 -o $OUT/track python scripts/run_track.py > $OUT/ncu_track.log 2>&1
$FULL -k regex:td3_update -s 1 -c 1 -o $OUT/td3 python scripts/run_td3.py > $OUT/ncu_td3.log 2>&1
$FULL -k regex:stats_finalize -c 1 -o $OUT/finalize python bench.py --steps 1 --warmup 0 --no-secondary --no-cpu-baseline --T 10 > $OUT/ncu_fin.log 2>&1
ls $OUT
