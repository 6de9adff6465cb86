#!/bin/bash
# TD3 A/B: bench td3_update value for each scripts/dbg/libl2f_<tag>.so (alternating twice)
for rep in 1 2; do for t in "$@"; do
  cp scripts/dbg/libl2f_$t.so paper_2311_13081_b200/libl2f.so
  python - <<PY
import os, sys, torch, json
sys.path.insert(0, os.getcwd())
import bench, inputs, paper_2311_13081_b200 as pkg
PY
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['modes']['td3_update']; print('$t', t['value'], t['roofline']['frac'])"
done; done
