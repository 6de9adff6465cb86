#!/bin/bash
# The compute-sanitizer substitute (the tool is closed on the measurement pool): the
# -DL2F_DEBUG_CHECKS build (bounds checks on every global / shared / tensor-memory index,
# bounded mbarrier waits, trap on failure) runs the whole GPU test suite and the small
# every-kernel invocation at several ragged sizes.  Usage (under gpurun): bash scripts/debug_checks.sh <tag>
set -u
OUT=gpurun_out/debug_checks_${1:-r2}
mkdir -p $OUT
export L2F_LIB_PATH=$PWD/build/ab/libl2f_debug.so
[ -f $L2F_LIB_PATH ] || { echo "build it first: scripts/build_variant.sh debug -DL2F_DEBUG_CHECKS"; exit 1; }
for n in 1 127 1000 4096; do
  L2F_SAN_N=$n timeout 600 python scripts/sanitize_run.py > $OUT/run_n$n.log 2>&1
  echo "every-kernel run N=$n rc=$? $(tail -1 $OUT/run_n$n.log)"
done
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1
echo "pytest -m gpu (debug build) rc=$? $(tail -1 $OUT/pytest_gpu.log)"
grep -h "L2F_CHECK failed" $OUT/*.log | sort | uniq -c | head
