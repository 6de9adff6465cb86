#!/bin/bash
# Profiling pass (run under gpurun on one B200).  Usage: scripts/profile.sh <tag>
# 1. plain run of the bench command (must exit 0 before any ncu run)
# 2. launch list of the same command (gpu__time_duration, serialised, cold cache)
# 3. ncu --set full on the dominant kernels (short variants of the same launches)
set -u
TAG=${1:-r1}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rollout_mlp -c 1 -o $OUT/mlp \
    python bench.py --steps 1 --warmup 0 --no-secondary --no-cpu-baseline --T 100 > $OUT/ncu_mlp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 10 -c 1 -o $OUT/step \
    python scripts/run_step.py > $OUT/ncu_step.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rollout_open -c 1 -o $OUT/open \
    python scripts/run_open.py > $OUT/ncu_open.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:track_mlp -c 1 -o $OUT/track \
    python scripts/run_track.py > $OUT/ncu_track.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:td3_update -s 1 -c 1 -o $OUT/td3 \
    python scripts/run_td3.py > $OUT/ncu_td3.log 2>&1
echo done
