"""Timings of the actor-MLP kernel family: C5 rollout (2^21 x 300), C4 (2^20 x 300), the
DR rollout (C5 + domain randomisation, 2^21 x 300) and Lissajous tracking (2^20 x 300):
env-steps/s of each, one line."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs
import paper_2311_13081_b200 as pkg

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
pol = pkg.Policy(inputs.policy_weights(146, 64, seed=7, out_bias=inputs.hover_policy_bias()))


def timed(fn, units):
    fn()
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return units / (e0.elapsed_time(e1) / 1e3)


out = {}
T = 300
for name, cfg, n in (("c5", inputs.config_c5(), 1 << 21), ("c4", inputs.config_c4(), 1 << 20),
                     ("c5_dr", dict(inputs.config_c5(), flags=inputs.config_c5()["flags"] | inputs.DOMAIN_RAND), 1 << 21)):
    env = pkg.Env(cfg, n)
    env.reset()
    out[name] = timed(lambda: env.rollout(T, policy=pol), n * T)
    del env
    torch.cuda.empty_cache()
n = 1 << 20
env = pkg.Env(inputs.config_c4(), n)
ct = torch.tensor([15.0, 5.5, 3.5], device="cuda").repeat(n // 3 + 1)[:n].contiguous()
out["track"] = timed(lambda: env.track(pol, ct, T), n * T)
print(" ".join("%s %.4g" % kv for kv in out.items()))
