#!/bin/bash
# ncu --set full of the C3 l2f_step kernel (specialised build).  Usage: bash scripts/prof_step.sh <tag>
OUT=gpurun_out/prof_${1:-r2}
mkdir -p $OUT
python scripts/run_step.py > $OUT/plain_step.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 10 -c 1 -o $OUT/step python scripts/run_step.py > $OUT/ncu_step.log 2>&1
