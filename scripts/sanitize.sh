#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over every kernel (one B200).
# Usage (under gpurun): bash scripts/sanitize.sh <tag>  -> gpurun_out/sanitize_<tag>/*.log
set -u
OUT=gpurun_out/sanitize_${1:-r2}
mkdir -p $OUT
python scripts/sanitize_run.py > $OUT/plain.log 2>&1 || { echo "plain run failed"; tail $OUT/plain.log; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  [ $tool = initcheck ] && extra="--track-unused-memory no"
  timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 python scripts/sanitize_run.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/$tool.log | tail -1)"
done
