#!/bin/bash
# C3 step-kernel A/B: us per l2f_step at 2^20 envs for each scripts/dbg/libl2f_<tag>.so
for t in "$@"; do
  cp scripts/dbg/libl2f_$t.so paper_2311_13081_b200/libl2f.so
  python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import inputs, paper_2311_13081_b200 as pkg
n = 1 << 20
env = pkg.Env(inputs.config_c3(), n); env.reset()
acts = [torch.tensor(inputs.actions_near_hover(1, n, seed=100 + k)[0], dtype=torch.float32, device="cuda") for k in range(8)]
o = env.make_out(obs_core=True, reward=True, flags=True)
for k in range(20): env.step(acts[k % 8], o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(400): env.step(acts[k % 8], o)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("T", ""), "%.2f us" % (e0.elapsed_time(e1) / 400 * 1e3))
PY
done
