#!/bin/bash
# open-loop A/B (C1 64x500 Philox, paper shape 8192 x 200k, dyn 2^20 x 1000) of build/ab/libl2f_<tag>.so
for t in "$@"; do
  cp build/ab/libl2f_$t.so paper_2311_13081_b200/libl2f.so
  python - <<PY
import sys, torch; sys.path.insert(0, ".")
import inputs, paper_2311_13081_b200 as pkg
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = []
for n, T in ((64, 500), (8192, 200000), (1 << 20, 1000)):
    env = pkg.Env(inputs.config_c1(), n); env.reset(); env.rollout(100); torch.cuda.synchronize()
    e0.record(); env.rollout(T); e1.record(); torch.cuda.synchronize()
    res.append("%d x %d: %.4g env-steps/s" % (n, T, n * T / (e0.elapsed_time(e1) / 1e3)))
print("$t", " | ".join(res))
PY
done
