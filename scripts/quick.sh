#!/bin/bash
# Quick perf check under gpurun: main bench line + secondary modes (no CPU baseline), compact.
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/quick.json 2> gpurun_out/quick.err || { tail -20 gpurun_out/quick.err; exit 1; }
python - <<'PY'
import json
d = json.loads(open("gpurun_out/quick.json").read().strip().splitlines()[-1])
print("mlp %.4g env-steps/s  frac %.3f  ms %.2f" % (d["value"], d["roofline"]["frac"], d["ms_per_step"]))
for k, v in d["modes"].items():
    rf = v.get("roofline", {})
    print(k, "%.4g" % v["value"], v["unit"], "frac %.3f" % rf["frac"] if rf else "", v.get("us_per_step", v.get("ms", v.get("ms_per_call", ""))))
PY
