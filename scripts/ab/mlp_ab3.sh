#!/bin/bash
# MLP-rollout A/B with longer timed regions: bench value (10 steps) for each build/ab/libl2f_<tag>.so,
# alternating three times
for rep in 1 2 3; do
for t in "$@"; do
  cp build/ab/libl2f_$t.so paper_2311_13081_b200/libl2f.so
  python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$t', d['value'])"
done
done
