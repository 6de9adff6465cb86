"""l2f_track workload for profiling: 2^20 envs x 100 steps, cycle times 15/5.5/3.5 s, C4 actor."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs
import paper_2311_13081_b200 as pkg

n = 1 << 20
env = pkg.Env(inputs.config_c4(), n)
pol = pkg.Policy(inputs.policy_weights(146, 64, seed=7, out_bias=inputs.hover_policy_bias()))
ct = torch.tensor([15.0, 5.5, 3.5], device="cuda").repeat(n // 3 + 1)[:n].contiguous()
env.track(pol, ct, 100)
torch.cuda.synchronize()
print("ok")
