#!/bin/bash
# Fast perf check of the headline kernel under gpurun: main bench line only (T = 1000, 2^21 envs).
python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/qm.json 2> gpurun_out/qm.err || { tail -20 gpurun_out/qm.err; exit 1; }
python - <<'PY'
import json
d = json.loads(open("gpurun_out/qm.json").read().strip().splitlines()[-1])
print("mlp %.4g env-steps/s  frac %.3f  ms %.2f  clk %s" % (d["value"], d["roofline"]["frac"], d["ms_per_step"], d["clocks"]["sm_mhz"]))
PY
