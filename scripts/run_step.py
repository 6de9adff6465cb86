"""C3 single-step workload for profiling: 2^20 envs, DR, l2f_step x 30."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs
import paper_2311_13081_b200 as pkg

n = 1 << 20
env = pkg.Env(inputs.config_c3(), n)
env.reset()
acts = [torch.tensor(inputs.actions_near_hover(1, n, seed=100 + k)[0], dtype=torch.float32, device="cuda") for k in range(8)]
o = env.make_out(obs_core=True, reward=True, flags=True)
for k in range(30):
    env.step(acts[k % 8], o)
torch.cuda.synchronize()
print("ok")
