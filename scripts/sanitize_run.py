"""Small invocation of every kernel of libl2f.so for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): N <= 4096 envs.  Usage: compute-sanitizer --tool <t> python scripts/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import inputs
import paper_2311_13081_b200 as pkg

dev = torch.device("cuda")
n = int(os.environ.get("L2F_SAN_N", "1000"))  # ragged: not a multiple of the 128-env tiles
for cfg in (inputs.config_c5(), inputs.config_c3()):
    env = pkg.Env(cfg, n)
    out = env.make_out(obs_core=True, reward=True, flags=True, final_state=True, obs_dense=True)
    env.reset(out=out)
    acts = torch.rand(4, n, device=dev) * 2 - 1
    for _ in range(3):
        env.step(acts, out)
    mask = (torch.arange(n, device=dev) % 3 == 0).to(torch.uint8)
    env.reset(mask=mask, out=out)
    env.rollout(8)  # open loop, Philox actions
    env.rollout(4, actions=torch.rand(4, 4, n, device=dev) * 2 - 1, trace_ids=torch.arange(0, n, 97, device=dev))
    W = inputs.policy_weights(146, 64, seed=7, out_bias=inputs.hover_policy_bias())
    pol = pkg.Policy(W)
    env.rollout(12, policy=pol, trace_ids=torch.arange(0, n, 131, device=dev))
    st = env.episode_stats(reset=True)
    env.recompute_rewards(0, torch.rand(17, 777, device=dev), torch.rand(4, 777, device=dev))
    a = pkg.policy_forward(pol, torch.rand(n, 146, device=dev))
    r = env.track(pol, 5.5, 10)
    torch.cuda.synchronize()
A, B, I = 2, 32, 146
td3 = pkg.TD3(A, I, B)
td3.params.uniform_(-0.1, 0.1)
o = td3.offsets()
td3.params[:, o["m_actor"]:].zero_()
g = torch.Generator(device=dev).manual_seed(0)
bt = {"o_a": torch.randn(A, B, I, device=dev, generator=g), "o_c": torch.randn(A, B, 28, device=dev, generator=g),
      "a": torch.rand(A, B, 4, device=dev, generator=g), "r": torch.randn(A, B, device=dev, generator=g),
      "o_a2": torch.randn(A, B, I, device=dev, generator=g), "o_c2": torch.randn(A, B, 28, device=dev, generator=g),
      "done": torch.zeros(A, B, device=dev), "eps": torch.randn(A, B, 4, device=dev, generator=g)}
td3.update(bt, update_actor=True)
torch.cuda.synchronize()
print("sanitize run ok, launches", pkg.launch_count())
