"""Throughput vs problem size: the fused rollout (envs per GPU) and the TD3 update (agents)."""
import os, sys, json, subprocess
sys.path.insert(0, os.getcwd())
import torch, numpy as np
for n in (1 << 18, 1 << 19, 1 << 20, 1 << 21, 1 << 22):
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-secondary", "--no-cpu-baseline",
                        "--envs-per-gpu", str(n)], capture_output=True, text=True)
    d = json.loads(r.stdout.strip().splitlines()[-1])
    print("rollout envs", n, "%.4g env-steps/s" % d["value"], "frac %.3f" % d["roofline"]["frac"], flush=True)
import paper_2311_13081_b200 as pkg
dev = torch.device("cuda")
for A in (148, 296, 592, 1184):
    B, I = 256, 146
    td3 = pkg.TD3(A, I, B, device=dev)
    g = torch.Generator(device=dev).manual_seed(3)
    td3.params.uniform_(-0.1, 0.1, generator=g)
    o = td3.offsets()
    td3.params[:, o["m_actor"]:].zero_()
    bt = {"o_a": torch.randn(A, B, I, device=dev) * 0.5, "o_c": torch.randn(A, B, 28, device=dev) * 0.5,
          "a": torch.rand(A, B, 4, device=dev) * 2 - 1, "r": torch.randn(A, B, device=dev),
          "o_a2": torch.randn(A, B, I, device=dev) * 0.5, "o_c2": torch.randn(A, B, 28, device=dev) * 0.5,
          "done": (torch.rand(A, B, device=dev) < 0.1).float(), "eps": torch.randn(A, B, 4, device=dev)}
    for k in range(4):
        td3.update(bt, update_actor=(k % 2 == 1))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(20):
        td3.update(bt, update_actor=(k % 2 == 1))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print("td3 agents", A, "%.4g agent-updates/s" % (A / (ms * 1e-3)), "%.3f ms/call" % ms, flush=True)
