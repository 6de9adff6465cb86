#!/bin/bash
# Phase timing of the MLP rollout (debug build build/ab/libl2f_phase.so, -DL2F_PHASE_TIMING):
# swaps the debug library in (the box copy is scratch) and prints per-warp cycles per phase.
cp build/ab/libl2f_phase.so paper_2311_13081_b200/libl2f.so
python bench.py --steps 1 --warmup 0 --no-secondary --no-cpu-baseline --T 200 > gpurun_out/phase.log 2>&1
grep L2F_PHASE gpurun_out/phase.log > gpurun_out/phase.txt
python scripts/phase_summary.py gpurun_out/phase.txt ${PHASE_STEPS:-5600}
