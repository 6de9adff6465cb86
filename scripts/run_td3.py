"""TD3 update workload for profiling: 148 agents x batch 256, actor 146-64-64-4, 4 updates."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_13081_b200 as pkg

A, B, I = 148, 256, 146
td3 = pkg.TD3(A, I, B)
g = torch.Generator(device="cuda").manual_seed(3)
td3.params.uniform_(-0.1, 0.1, generator=g)
td3.params[:, td3.offsets()["m_actor"]:].zero_()
bt = {"o_a": torch.randn(A, B, I, device="cuda", generator=g) * 0.5, "o_c": torch.randn(A, B, 28, device="cuda", generator=g) * 0.5,
      "a": torch.rand(A, B, 4, device="cuda", generator=g) * 2 - 1, "r": torch.randn(A, B, device="cuda", generator=g),
      "o_a2": torch.randn(A, B, I, device="cuda", generator=g) * 0.5, "o_c2": torch.randn(A, B, 28, device="cuda", generator=g) * 0.5,
      "done": (torch.rand(A, B, device="cuda", generator=g) < 0.1).float(), "eps": torch.randn(A, B, 4, device="cuda", generator=g)}
for k in range(4):
    td3.update(bt, update_actor=(k % 2 == 1))
torch.cuda.synchronize()
print("ok")
