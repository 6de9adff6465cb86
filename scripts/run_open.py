"""Open-loop rollouts for profiling (Philox random actions).
  python scripts/run_open.py dyn   C1 flags (dynamics only, the paper-comparable mode): 2^20 envs x 1000 steps
  python scripts/run_open.py c5    C5 features: 2^21 envs x 200 steps"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs
import paper_2311_13081_b200 as pkg

mode = sys.argv[1] if len(sys.argv) > 1 else "dyn"
cfg, n, T = (inputs.config_c1(), 1 << 20, 1000) if mode == "dyn" else (inputs.config_c5(), 1 << 21, 200)
env = pkg.Env(cfg, n)
env.reset()
env.rollout(T)
torch.cuda.synchronize()
print("ok")
