"""C3 l2f_step timing (2^20 envs, DR, ring of 8 action buffers): us per step over 400 steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs
import paper_2311_13081_b200 as pkg

n = int(os.environ.get("L2F_N", 1 << 20))
env = pkg.Env(inputs.config_c3(), n)
env.reset()
acts = [torch.tensor(inputs.actions_near_hover(1, n, seed=100 + k)[0], dtype=torch.float32, device="cuda") for k in range(8)]
o = env.make_out(obs_core=True, reward=True, flags=True)
for k in range(40):
    env.step(acts[k % 8], o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(400):
    env.step(acts[k % 8], o)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 400 * 1e3
print("step_us %.2f n %d ns_per_kenv %.3f" % (us, n, us / n * 1e6))
