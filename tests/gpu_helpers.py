"""Helpers for the GPU <-> oracle parity tests: moving env state between the CUDA env's SoA
workspace and the oracle's per-env records, and the tolerances of BASELINE north_star."""
from __future__ import annotations

import numpy as np
import torch

import oracle

# north_star: single step per-component |err| <= 1e-5 |x| + 1e-6
REL, ABS = 1e-5, 1e-6


def close(gpu, ref, rel=REL, abs_=ABS):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return np.abs(gpu - ref) <= rel * np.abs(ref) + abs_


def close_step(gpu, ref, prev, rel=REL, abs_=ABS):
    """Single-step tolerance with the component's scale over the step (Q27):
    |err| <= 1e-5 max(|x_t|, |x_t+1|) + 1e-6.  FP32 carries ~eps |dx| absolute error on a
    component that changes by dx in one step, so a value landing near zero after a large
    change is judged against the change's scale."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = np.maximum(np.abs(ref), np.abs(np.asarray(prev, dtype=np.float64)))
    return np.abs(gpu - ref) <= rel * scale + abs_


# obs_core index -> state index whose pre-step value sets the scale (p, v, omega blocks)
OBS_PREV = {0: 0, 1: 1, 2: 2, 12: 7, 13: 8, 14: 9, 15: 10, 16: 11, 17: 12}


def close_obs(gpu_obs, ref_obs, s_prev):
    prev = np.zeros(len(ref_obs))
    for j, k in OBS_PREV.items():
        prev[j] = s_prev[k]
    return close_step(gpu_obs, ref_obs, prev)


def snapshot(env, cols=None) -> dict:
    """Component-major copies of the env arrays; cols: only these env columns (full-size runs)."""
    torch.cuda.synchronize()
    out = {}
    for k in ("state", "dist", "dr", "hist", "hist_t0", "hist_fill", "ep_step", "ep_return"):
        x = getattr(env, k).detach()
        if cols is not None:
            x = x[..., torch.as_tensor(np.asarray(cols), device=x.device)]
        out[k] = x.cpu().numpy().copy()
    return out


def load_snapshot(env, snap: dict):
    for k, v in snap.items():
        env.set_logical(k, v)
    torch.cuda.synchronize()


def logical_hist(snap: dict, i: int, t_next: int, n_hist: int) -> np.ndarray:
    """Most-recent-first history H[k] of env i when the next step is t_next (include/l2f.h):
    tau = t_next - 1 - k; ring slot (tau mod N_H) if tau >= hist_t0 else hist_fill."""
    out = np.zeros((n_hist, 4))
    t0 = int(snap["hist_t0"][i])
    for k in range(n_hist):
        tau = t_next - 1 - k
        out[k] = snap["hist"][tau % n_hist, :, i] if tau >= t0 else snap["hist_fill"][:, i]
    return out


def to_oracle(snap: dict, idx, t: int, n_hist: int) -> np.ndarray:
    """GPU SoA workspace -> oracle records (H[k] = a_{t-1-k}, most recent first)."""
    idx = np.asarray(idx)
    E = oracle.new_envs(len(idx))
    for j, i in enumerate(idx):
        E[j]["s"] = snap["state"][:, i]
        E[j]["dist"] = snap["dist"][:, i]
        E[j]["dr"] = snap["dr"][:, i]
        if n_hist:
            E[j]["hist"][:n_hist] = logical_hist(snap, i, t, n_hist)
        E[j]["ep_step"] = snap["ep_step"][i]
        E[j]["ep_return"] = snap["ep_return"][i]
    return E


def near_threshold(so, cfg, extra: float = 0.0) -> bool:
    """Q22: an env-step whose termination margin is within the compared tolerance."""
    thr = (cfg["term_pos"], cfg["term_vel"], cfg["term_angvel"])
    for m, t in zip(so.margin, thr):
        if abs(m) <= max(1e-6, REL * abs(t) + ABS) + extra:
            return True
    return False


class TolStats:
    """Accounting of the two single-step tolerance readings (Q27, Q36).

    Every compared value is first judged by north_star's bound |err| <= 1e-5 |x| + 1e-6 on the
    oracle's value x; a value that misses it must meet the widened bound of its reading, and is
    counted.  State components (Q27): 1e-5 max(|x_t|, |x_t+1|) + 1e-6.  Rewards: the tests
    require zero widened rewards (north_star's bound holds for every reward measured); the
    scale S = 2 sum_k |term_k| of the reward's terms on s' is only reported for a failure.
    Tests bound the widened fraction (round-2 measurement: <= 8 of 170 000 state components,
    all body rates), so the reading cannot silently absorb a real discrepancy."""

    def __init__(self):
        self.n_state = self.w_state = self.n_rew = self.w_rew = 0
        self.examples = []

    def state(self, gpu, ref, prev, tag=None) -> bool:
        strict = close(gpu, ref)
        wide = close_step(gpu, ref, prev)
        self.n_state += strict.size
        k = int(np.count_nonzero(~strict & wide))
        self.w_state += k
        if k and len(self.examples) < 8:
            self.examples.append((tag, np.flatnonzero(~strict & wide).tolist()))
        return bool(np.all(wide))

    def reward(self, gpu, ref, scale) -> bool:
        self.n_rew += 1
        if close(gpu, ref):
            return True
        self.w_rew += 1
        return abs(float(gpu) - float(ref)) <= REL * scale + ABS

    def summary(self) -> dict:
        return {"state_components": self.n_state, "state_widened": self.w_state,
                "state_widened_frac": self.w_state / max(self.n_state, 1), "rewards": self.n_rew,
                "rewards_widened": self.w_rew, "rewards_widened_frac": self.w_rew / max(self.n_rew, 1),
                "examples": self.examples}

    def report(self, name: str):
        import json
        import os
        d = os.environ.get("L2F_TOLSTATS_DIR")
        if d:
            os.makedirs(d, exist_ok=True)
            with open(os.path.join(d, name + ".json"), "w") as f:
                json.dump(self.summary(), f, indent=1)
        print(name, self.summary())


def reward_scale(cfg, t, s1, a) -> float:
    """Q36 scale S = 2 sum |term| of the reward at stage t, state s1, action a:
    a tolerance scale only (the parity value itself is the oracle's reward)."""
    w, _ = oracle.stage(cfg, t)
    s1 = np.asarray(s1, dtype=np.float64)
    a = np.asarray(a, dtype=np.float64)
    rab = np.array(list(w.C_rab))
    terms = [w.C_rs, w.C_rp * np.sum(s1[0:3] ** 2), w.C_rq * abs(1 - s1[3] ** 2), w.C_rv * np.sum(s1[7:10] ** 2),
             w.C_rw * np.sum(s1[10:13] ** 2), w.C_ra * np.sum((a - rab) ** 2)]
    return 2.0 * float(np.sum(np.abs(terms)))
