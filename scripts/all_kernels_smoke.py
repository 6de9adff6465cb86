"""Small, ragged invocations of every kernel in one process (odd sizes, traces, all outputs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs
import paper_2311_13081_b200 as pkg

n = 3 * 128 + 45
env = pkg.Env(inputs.config_c3(), n)
env.reset()
o = env.make_out(obs_core=True, reward=True, flags=True, obs_dense=True, obs_critic=True, final_state=True)
for k in range(3):
    env.step(torch.rand(4, n, device="cuda") * 2 - 1, o)
env.rollout(5)
pol = pkg.Policy(inputs.policy_weights(146, 64, seed=5, out_bias=inputs.hover_policy_bias()))
env5 = pkg.Env(inputs.config_c5(), n)
env5.reset()
env5.rollout(6, policy=pol, trace_ids=torch.tensor([0, 7, n - 1]))
env5.track(pol, 5.5, 4)
pkg.policy_forward(pol, torch.randn(300, 146, device="cuda"))
env5.episode_stats()
td3 = pkg.TD3(2, 146, 37)
td3.params.uniform_(-0.1, 0.1)
o_ = td3.offsets()
td3.params[:, o_["m_actor"]:].zero_()
bt = {"o_a": torch.randn(2, 37, 146), "o_c": torch.randn(2, 37, 28), "a": torch.rand(2, 37, 4), "r": torch.randn(2, 37),
      "o_a2": torch.randn(2, 37, 146), "o_c2": torch.randn(2, 37, 28), "done": torch.zeros(2, 37), "eps": torch.randn(2, 37, 4)}
td3.update(bt, update_actor=True)
td3.actor_policy(1)
torch.cuda.synchronize()
print("all kernels ok")
