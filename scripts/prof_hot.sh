#!/bin/bash
# ncu --set full captures of the two hot kernels (fused MLP rollout at T=100, l2f_step at C3).
# Usage (under gpurun): bash scripts/prof_hot.sh <tag>
set -u
TAG=${1:-r2}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
python bench.py --steps 1 --warmup 0 --no-secondary --no-cpu-baseline --T 100 > $OUT/plain.log 2>&1 || { echo "plain run failed"; tail $OUT/plain.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:rollout_mlp -c 1 -o $OUT/mlp \
    python bench.py --steps 1 --warmup 0 --no-secondary --no-cpu-baseline --T ${MLP_T:-1000} > $OUT/ncu_mlp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 10 -c 1 -o $OUT/step \
    python scripts/run_step.py > $OUT/ncu_step.log 2>&1
echo done
