"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic: only literal configuration values
(BASELINE.json configs), seeded random arrays and packing of those
arrays into the layouts each side's binding expects.  Both ``oracle/`` and the CUDA binding
consume these inputs; neither side's arithmetic lives here.

Config dict schema (one dict per environment batch; both bindings marshal it):
  flags, n_hist, max_episode_steps, seed, dt, params{...}, dr_range, init_pos, init_angle,
  init_vel, init_angvel, init_rpm, dist_force, dist_torque, obs_sigma[4], term_pos, term_vel,
  term_angvel, curriculum{init, target, factor, sigma_init, sigma_target, sigma_factor, interval}
"""
from __future__ import annotations

import copy
import math

import numpy as np

OBS_NOISE, ACTION_NOISE, TERMINATION, AUTO_RESET, DISTURBANCE, DOMAIN_RAND = (1, 2, 4, 8, 16, 32)
NO_ROTOR_DELAY = 64  # ablation switch (Table II "Rotor Delay")
ALL_NO_DR = OBS_NOISE | ACTION_NOISE | TERMINATION | AUTO_RESET | DISTURBANCE

# Crazyflie 2.1-style defaults.  Paper values: m = 27 g, T_m = 0.15 s, dt = 0.01 s
# (P:165).  Everything else is SURVEY.md Appendix A (documented defaults; the paper's
# parameter PDF, is absent).  No parity test depends on these particular values.
_L = 0.028
CRAZYFLIE = {
    "mass": 0.027,
    "J": [3.85e-6, 3.85e-6, 5.9675e-6],
    "rotor_pos": [[_L, -_L, 0.0], [-_L, -_L, 0.0], [-_L, _L, 0.0], [_L, _L, 0.0]],
    "spin_dir": [-1.0, 1.0, -1.0, 1.0],
    "thrust_c": [0.0, 0.0, 3.16e-10],
    "torque_c": 0.005964552,
    "motor_tau": 0.15,
    "rpm_min": 0.0,
    "rpm_max": 21702.0,
    "gravity": 9.81,
}
# Normalised hover action for CRAZYFLIE (0.33405).  A literal used only
# to shape synthetic inputs (near-hover action streams, C_rab, the policy's output bias).
A_HOVER = 0.33405

_W_INIT = {"C_rp": 1.0, "C_rq": 1.0, "C_rv": 0.05, "C_rw": 0.005, "C_ra": 0.01,
           "C_rab": [A_HOVER] * 4, "C_rs": 1.0}
_W_TARGET = {"C_rp": 4.0, "C_rq": 1.0, "C_rv": 0.05, "C_rw": 0.005, "C_ra": 0.5,
             "C_rab": [A_HOVER] * 4, "C_rs": 1.0}
_W_FACTOR = {"C_rp": 1.2, "C_rq": 1.0, "C_rv": 1.0, "C_rw": 1.0, "C_ra": 1.4,
             "C_rab": [1.0] * 4, "C_rs": 1.0}


def base_config(**over) -> dict:
    cfg = {
        "flags": ALL_NO_DR,
        "n_hist": 32,
        "max_episode_steps": 500,
        "seed": 0x5EED_1234_ABCD,
        "dt": 0.01,
        "params": copy.deepcopy(CRAZYFLIE),
        "dr_range": [0.8, 1.2],
        "init_pos": 0.3,
        "init_angle": math.pi / 2,
        "init_vel": 1.0,
        "init_angvel": 1.0,
        "init_rpm": [CRAZYFLIE["rpm_min"], CRAZYFLIE["rpm_max"]],
        "dist_force": 0.0265,
        "dist_torque": 1e-5,
        "obs_sigma": [0.002, 0.01, 0.02, 0.1],
        "term_pos": 0.6,
        "term_vel": 10.0,
        "term_angvel": 35.0,
        "curriculum": {
            "init": copy.deepcopy(_W_INIT),
            "target": copy.deepcopy(_W_TARGET),
            "factor": copy.deepcopy(_W_FACTOR),
            "sigma_init": 0.1,
            "sigma_target": 0.02,
            "sigma_factor": 0.8,
            "interval": 100000,
        },
    }
    for k, v in over.items():
        cfg[k] = v
    return cfg


# The five BASELINE.json configs.
def config_c1(**over) -> dict:
    """64 envs x 500 steps, fixed params, open-loop random actions, no noise/resets."""
    d = dict(flags=0, max_episode_steps=0, seed=1)
    d.update(over)
    return base_config(**d)


def config_c2(**over) -> dict:
    """4096 envs x 1000 steps, obs/action noise, reward, termination, auto-reset."""
    d = dict(flags=ALL_NO_DR, seed=2)
    d.update(over)
    return base_config(**d)


def config_c3(**over) -> dict:
    """2^20 envs, per-env DR of mass/inertia/thrust, single-step API."""
    d = dict(flags=ALL_NO_DR | DOMAIN_RAND, seed=3)
    d.update(over)
    return base_config(**d)


def config_c4(**over) -> dict:
    """2^20 envs x 1000 steps fused MLP rollout, N_H = 32."""
    d = dict(flags=ALL_NO_DR, seed=4)
    d.update(over)
    return base_config(**d)


def config_c5(**over) -> dict:
    """2^24 envs over 8 GPUs, fused rollout + curriculum (4 stages in 1000 steps) + stats."""
    d = dict(flags=ALL_NO_DR, seed=5)
    d.update(over)
    cfg = base_config(**d)
    cfg["curriculum"]["interval"] = 250
    return cfg


CONFIG_SIZES = {"C1": (64, 500), "C2": (4096, 1000), "C3": (1 << 20, 1),
                "C4": (1 << 20, 1000), "C5": (1 << 24, 1000)}


# ----------------------------------------------------------------------------------------
# seeded arrays
# ----------------------------------------------------------------------------------------
def actions_uniform(T: int, n: int, seed: int = 11) -> np.ndarray:
    """Open-loop random RPM actions, literally U(-1,1) of shape (T, 4, n)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (T, 4, n))


def actions_near_hover(T: int, n: int, seed: int = 12, sigma: float = 0.2) -> np.ndarray:
    """a_hover + sigma N(0,1), clipped to [-1,1], shape (T, 4, n)."""
    a = A_HOVER + sigma * np.random.default_rng(seed).standard_normal((T, 4, n))
    return np.clip(a, -1.0, 1.0)


def random_states(n: int, seed: int = 21, params: dict | None = None) -> dict:
    """Random valid states for single-step parity (unit quaternions, rotor speeds in range,
    positions/velocities inside the termination box).  Returns SoA arrays."""
    p = params or CRAZYFLIE
    g = np.random.default_rng(seed)
    q = g.standard_normal((4, n))
    q /= np.linalg.norm(q, axis=0, keepdims=True)
    s = np.zeros((17, n))
    s[0:3] = g.uniform(-0.5, 0.5, (3, n))
    s[3:7] = q
    s[7:10] = g.uniform(-3, 3, (3, n))
    s[10:13] = g.uniform(-10, 10, (3, n))
    s[13:17] = g.uniform(p["rpm_min"], p["rpm_max"], (4, n))
    dist = np.concatenate([g.uniform(-0.0265, 0.0265, (3, n)), g.uniform(-1e-5, 1e-5, (3, n))])
    dr = g.uniform(0.8, 1.2, (5, n))
    hist = g.uniform(-1, 1, (32, 4, n))
    ep_step = g.integers(0, 500, n).astype(np.int32)
    ep_return = g.uniform(-50, 50, n)
    return {"state": s, "dist": dist, "dr": dr, "hist": hist, "ep_step": ep_step,
            "ep_return": ep_return}


def policy_weights(in_dim: int = 146, hidden: int = 64, seed: int = 7,
                   out_bias: float | None = None) -> dict:
    """Actor MLP in_dim -> hidden -> hidden -> 4 with U(+-1/sqrt(fan_in)) init (Q21), as fp16
    bit patterns (uint16), row-major [out][in].  out_bias: fill b3 (e.g. atanh(A_HOVER) so the
    random policy roughly hovers)."""
    g = np.random.default_rng(seed)

    def lin(o, i):
        b = 1.0 / math.sqrt(i)
        return g.uniform(-b, b, (o, i)), g.uniform(-b, b, (o,))

    W1, b1 = lin(hidden, in_dim)
    W2, b2 = lin(hidden, hidden)
    W3, b3 = lin(4, hidden)
    if out_bias is not None:
        b3 = np.full(4, out_bias)
    f16 = lambda a: np.asarray(a, dtype=np.float16).view(np.uint16)  # noqa: E731
    return {"W1": f16(W1), "b1": f16(b1), "W2": f16(W2), "b2": f16(b2), "W3": f16(W3), "b3": f16(b3)}


def hover_policy_bias() -> float:
    return float(np.arctanh(A_HOVER))


def trace_ids(n_envs: int, k: int, seed: int = 31) -> np.ndarray:
    """K distinct env indices spread over [0, n_envs) for traced parity."""
    g = np.random.default_rng(seed)
    return np.sort(g.choice(n_envs, size=min(k, n_envs), replace=False)).astype(np.int64)
