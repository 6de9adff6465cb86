"""C3 l2f_step (2^20 envs, DR): us per step from stream launches and from a CUDA graph of 50
steps (8 action buffers in rotation)."""
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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for k in range(20):
        env.step(acts[k % 8], o)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
e0.record()
for k in range(400):
    env.step(acts[k % 8], o)
e1.record()
torch.cuda.synchronize()
plain = e0.elapsed_time(e1) / 400 * 1e3
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for k in range(50):
        env.step(acts[k % 8], o)
g.replay()
torch.cuda.synchronize()
e0.record()
for r in range(8):
    g.replay()
e1.record()
torch.cuda.synchronize()
graph = e0.elapsed_time(e1) / 400 * 1e3
print("step_us plain %.2f graph %.2f" % (plain, graph))
