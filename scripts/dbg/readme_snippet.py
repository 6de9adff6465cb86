import torch, inputs, paper_2311_13081_b200 as l2f
env = l2f.Env(inputs.config_c4(), 1 << 20)          # 2^20 envs resident in HBM
env.reset()
pol = l2f.Policy(inputs.policy_weights(146, 64))    # fp16 actor 146-64-64-4
env.rollout(1000, policy=pol)                       # one fused tcgen05 launch
print(env.episode_stats())                          # FP64 episode statistics
r = env.track(pol, torch.tensor([15.0, 5.5, 3.5], device="cuda").repeat(env.n // 3 + 1)[:env.n], 550)
print(r["rmse"].mean(), (r["steps_ok"] == 550).float().mean())
td3 = l2f.TD3(n_agents=148, in_dim=146, batch=256)
B = {k: torch.randn(148, 256, d, device="cuda") * 0.3 for k, d in (("o_a", 146), ("o_c", 28), ("o_a2", 146), ("o_c2", 28), ("eps", 4))}
B["a"] = torch.rand(148, 256, 4, device="cuda") * 2 - 1
B["r"] = torch.randn(148, 256, device="cuda"); B["done"] = (torch.rand(148, 256, device="cuda") < 0.1).float()
print(td3.update(B, update_actor=True)[:2])
print("readme ok")
