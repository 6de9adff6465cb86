#!/bin/bash
# A/B of whole-library builds: MLP rollout, C3 step, TD3 values per build/ab/libl2f_<tag>.so
for rep in 1 2; do for t in "$@"; do
  cp build/ab/libl2f_$t.so paper_2311_13081_b200/libl2f.so
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['modes']; print('$t', '%.4g' % d['value'], '%.2f us' % m['C3_step_api']['us_per_step'], '%.4g' % m['td3_update']['value'], '%.4g' % m['open_loop_dynamics']['value'], '%.4g' % m['lissajous_tracking']['value'])"
done; done
