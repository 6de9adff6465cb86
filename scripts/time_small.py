"""C1 / C2 latency-bound timings (bench.py small_configs): us per step of the open-loop rollout
and of l2f_step replayed from a CUDA graph."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import inputs
import paper_2311_13081_b200 as pkg

out = bench.small_configs(pkg, inputs, torch, torch.device("cuda:0"))
print(" ".join("%s %.3f" % (k, v["us_per_step"]) for k, v in out.items()))
