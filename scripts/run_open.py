"""Open-loop C2-feature rollout for profiling: 2^20 envs x 100 steps, Philox random actions."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs
import paper_2311_13081_b200 as pkg

n = 1 << 20
env = pkg.Env(inputs.config_c2(), n)
env.reset()
env.rollout(100)
torch.cuda.synchronize()
print("ok")
