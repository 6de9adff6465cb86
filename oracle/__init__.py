"""FP64 CPU oracle for the batched quadrotor environment step (arXiv 2311.13081).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs, never by the product package
(paper_2311_13081_b200).  It wraps ``l2f_oracle.c`` (plain scalar C, FP64) with ctypes and
shares no code with the CUDA path; only the seeded input generators in ``inputs/`` serve both.

The arithmetic lives in l2f_oracle.c, which cites PAPER.md per function.  This module only
marshals numpy arrays and config dicts into the oracle's own structs.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "l2f_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()

# flags / indices (mirrors of the C enums)
OBS_NOISE, ACTION_NOISE, TERMINATION, AUTO_RESET, DISTURBANCE, DOMAIN_RAND, NO_ROTOR_DELAY = (1, 2, 4, 8, 16, 32,
                                                                                   64)
FLAG_TERMINATED, FLAG_TRUNCATED, FLAG_DIVERGED, FLAG_RESET = 1, 2, 4, 8
STATS = ["episodes", "terminated", "truncated", "diverged", "sum_len", "sum_ret", "sum_ret_sq",
         "env_steps"]
TRACE_FIELDS = 28
MODE_ACTIONS, MODE_RANDOM, MODE_POLICY = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc -O2 (no fast-math, no intrinsics)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                                   "-ffp-contract=off", "-o", tmp, _SRC, "-lm", "-lpthread"])
            os.replace(tmp, _LIB)
    return _LIB


class Params(C.Structure):
    _fields_ = [("mass", C.c_double), ("J", C.c_double * 3), ("rotor_pos", (C.c_double * 3) * 4),
                ("spin_dir", C.c_double * 4), ("thrust_c", C.c_double * 3), ("torque_c", C.c_double),
                ("motor_tau", C.c_double), ("rpm_min", C.c_double), ("rpm_max", C.c_double),
                ("gravity", C.c_double)]


class Weights(C.Structure):
    _fields_ = [("C_rp", C.c_double), ("C_rq", C.c_double), ("C_rv", C.c_double),
                ("C_rw", C.c_double), ("C_ra", C.c_double), ("C_rab", C.c_double * 4),
                ("C_rs", C.c_double)]


class Config(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("n_hist", C.c_int32), ("max_episode_steps", C.c_int32),
                ("pad0", C.c_int32), ("seed", C.c_uint64), ("dt", C.c_double),
                ("nominal", Params), ("dr_lo", C.c_double), ("dr_hi", C.c_double),
                ("init_pos", C.c_double), ("init_angle", C.c_double), ("init_vel", C.c_double),
                ("init_angvel", C.c_double), ("init_rpm_lo", C.c_double), ("init_rpm_hi", C.c_double),
                ("dist_force", C.c_double), ("dist_torque", C.c_double),
                ("obs_sigma", C.c_double * 4), ("term_pos", C.c_double), ("term_vel", C.c_double),
                ("term_angvel", C.c_double), ("w_init", Weights), ("w_target", Weights),
                ("w_factor", Weights), ("sigma_init", C.c_double), ("sigma_target", C.c_double),
                ("sigma_factor", C.c_double), ("interval", C.c_int64)]


class StepOut(C.Structure):
    _fields_ = [("reward", C.c_double), ("flags", C.c_uint32), ("pad", C.c_uint32),
                ("a_applied", C.c_double * 4), ("final_s", C.c_double * 17),
                ("margin", C.c_double * 3)]


class Policy(C.Structure):
    _fields_ = [("in_dim", C.c_int32), ("hidden", C.c_int32),
                ("W1", C.c_void_p), ("b1", C.c_void_p), ("W2", C.c_void_p), ("b2", C.c_void_p),
                ("W3", C.c_void_p), ("b3", C.c_void_p)]


ENV_DTYPE = np.dtype([("s", "<f8", (17,)), ("dist", "<f8", (6,)), ("dr", "<f8", (5,)),
                      ("hist", "<f8", (32, 4)), ("ep_step", "<i8"), ("ep_return", "<f8")])

class TD3Hyper(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("gamma", "tau", "sigma_t", "clip_t", "lr_actor", "lr_critic", "beta1",
                                          "beta2", "eps")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        L.or_philox4x32_10.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.or_uniform.restype = C.c_double
        L.or_uniform.argtypes = [C.c_uint32]
        L.or_box_muller.argtypes = [C.c_uint32, C.c_uint32, dp]
        L.or_q16.restype = C.c_double
        L.or_q16.argtypes = [C.c_double]
        L.or_half_to_double.restype = C.c_double
        L.or_half_to_double.argtypes = [C.c_uint16]
        L.or_rotation.argtypes = [dp, dp]
        L.or_effective_params.argtypes = [C.POINTER(Config), dp, C.POINTER(Params)]
        L.or_derivative.argtypes = [C.POINTER(Params), dp, dp, dp, dp]
        L.or_rk4.argtypes = [C.POINTER(Params), dp, dp, dp, C.c_double, dp]
        L.or_project.argtypes = [C.POINTER(Params), dp]
        L.or_action_to_rpm.restype = C.c_double
        L.or_action_to_rpm.argtypes = [C.POINTER(Params), C.c_double]
        L.or_stage.argtypes = [C.POINTER(Config), C.c_int64, C.POINTER(Weights), dp]
        L.or_reward.restype = C.c_double
        L.or_reward.argtypes = [C.POINTER(Weights), dp, dp]
        L.or_reset.argtypes = [C.POINTER(Config), C.c_uint64, C.c_uint64, C.c_void_p]
        L.or_observe.argtypes = [C.POINTER(Config), C.c_void_p, C.c_uint64, C.c_uint64, dp]
        L.or_mlp.argtypes = [C.POINTER(Policy), dp, dp]
        L.or_critic_observe.argtypes = [C.c_void_p, dp]
        L.or_recompute_reward.restype = C.c_double
        L.or_recompute_reward.argtypes = [C.POINTER(Config), C.c_int64, dp, dp]
        L.or_mlp_min_midpoint_margin.restype = C.c_double
        L.or_mlp_min_midpoint_margin.argtypes = [C.POINTER(Policy), dp]
        L.or_env_step.argtypes = [C.POINTER(Config), C.c_void_p, C.c_uint64, C.c_uint64, dp,
                                  C.POINTER(StepOut), dp]
        L.or_random_action.argtypes = [C.POINTER(Config), C.c_uint64, C.c_uint64, dp]
        L.or_rollout.argtypes = [C.POINTER(Config), C.c_void_p, C.c_void_p, C.c_int64, C.c_uint64,
                                 C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, dp,
                                 C.c_int32]
        L.or_lissajous.argtypes = [C.c_double] * 5 + [dp, dp]
        L.or_shift_observation.argtypes = [dp, dp, dp, C.c_double, C.c_double]
        L.or_hover_rpm.restype = C.c_double
        L.or_hover_rpm.argtypes = [C.POINTER(Params)]
        L.or_track.argtypes = [C.POINTER(Config), C.c_void_p, C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                               C.c_double, C.c_double, C.c_double, C.c_double, C.c_int32, dp, dp,
                               C.POINTER(C.c_int32), C.c_void_p]
        L.or_net_size.restype = C.c_int64
        L.or_net_size.argtypes = [C.c_int32, C.c_int32, C.c_int32]
        L.or_td3_update.argtypes = [dp, C.c_int32, C.c_int32, dp, dp, dp, dp, dp, dp, dp, dp,
                                    C.POINTER(TD3Hyper), C.c_int64, C.c_int64, C.c_int32, dp, C.c_void_p]
        for f in ("or_sizeof_config", "or_sizeof_env", "or_sizeof_step_out"):
            getattr(L, f).restype = C.c_int64
        assert L.or_sizeof_config() == C.sizeof(Config), "oracle Config mirror out of sync"
        assert L.or_sizeof_env() == ENV_DTYPE.itemsize, "oracle env mirror out of sync"
        assert L.or_sizeof_step_out() == C.sizeof(StepOut), "oracle StepOut mirror out of sync"
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _d(x):
    return np.ascontiguousarray(x, dtype=np.float64)


# ----------------------------------------------------------------------------------------
# config marshalling (input dict -> oracle struct)
# ----------------------------------------------------------------------------------------
def _params(d) -> Params:
    p = Params()
    p.mass = d["mass"]
    for i in range(3):
        p.J[i] = d["J"][i]
        p.thrust_c[i] = d["thrust_c"][i]
    for i in range(4):
        for j in range(3):
            p.rotor_pos[i][j] = d["rotor_pos"][i][j]
        p.spin_dir[i] = d["spin_dir"][i]
    p.torque_c = d["torque_c"]
    p.motor_tau = d["motor_tau"]
    p.rpm_min = d["rpm_min"]
    p.rpm_max = d["rpm_max"]
    p.gravity = d["gravity"]
    return p


def _weights(d) -> Weights:
    w = Weights()
    for k in ("C_rp", "C_rq", "C_rv", "C_rw", "C_ra", "C_rs"):
        setattr(w, k, d[k])
    for i in range(4):
        w.C_rab[i] = d["C_rab"][i]
    return w


def config(d: dict) -> Config:
    c = Config()
    c.flags = int(d["flags"])
    c.n_hist = int(d["n_hist"])
    c.max_episode_steps = int(d["max_episode_steps"])
    c.seed = int(d["seed"])
    c.dt = d["dt"]
    c.nominal = _params(d["params"])
    c.dr_lo, c.dr_hi = d["dr_range"]
    c.init_pos, c.init_angle, c.init_vel = d["init_pos"], d["init_angle"], d["init_vel"]
    c.init_angvel = d["init_angvel"]
    c.init_rpm_lo, c.init_rpm_hi = d["init_rpm"]
    c.dist_force, c.dist_torque = d["dist_force"], d["dist_torque"]
    for i in range(4):
        c.obs_sigma[i] = d["obs_sigma"][i]
    c.term_pos, c.term_vel, c.term_angvel = d["term_pos"], d["term_vel"], d["term_angvel"]
    cur = d["curriculum"]
    c.w_init, c.w_target, c.w_factor = _weights(cur["init"]), _weights(cur["target"]), _weights(cur["factor"])
    c.sigma_init, c.sigma_target, c.sigma_factor = cur["sigma_init"], cur["sigma_target"], cur["sigma_factor"]
    c.interval = int(cur["interval"])
    return c


def params_struct(d: dict) -> Params:
    return _params(d)


def weights_struct(d: dict) -> Weights:
    return _weights(d)


# ----------------------------------------------------------------------------------------
# thin wrappers
# ----------------------------------------------------------------------------------------
def philox(ctr, key) -> np.ndarray:
    c = (C.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (C.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (C.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return np.array(list(o), dtype=np.uint32)


def uniform(x: int) -> float:
    return lib().or_uniform(int(x) & 0xFFFFFFFF)


def box_muller(xa: int, xb: int):
    z = np.zeros(2)
    lib().or_box_muller(int(xa) & 0xFFFFFFFF, int(xb) & 0xFFFFFFFF, _dp(z))
    return z


def q16(x) -> np.ndarray:
    L = lib()
    x = np.asarray(x, dtype=np.float64)
    return np.array([L.or_q16(float(v)) for v in x.ravel()]).reshape(x.shape)


def half_to_double(h) -> np.ndarray:
    L = lib()
    h = np.asarray(h, dtype=np.uint16)
    return np.array([L.or_half_to_double(int(v)) for v in h.ravel()]).reshape(h.shape)


def rotation(q) -> np.ndarray:
    R = np.zeros(9)
    lib().or_rotation(_dp(_d(q)), _dp(R))
    return R.reshape(3, 3)


def effective_params(cfg: dict, dr) -> Params:
    p = Params()
    c = config(cfg)
    lib().or_effective_params(C.byref(c), _dp(_d(dr)), C.byref(p))
    return p


def derivative(params: Params, s, u, dist) -> np.ndarray:
    ds = np.zeros(17)
    lib().or_derivative(C.byref(params), _dp(_d(s)), _dp(_d(u)), _dp(_d(dist)), _dp(ds))
    return ds


def rk4(params: Params, s, u, dist, h) -> np.ndarray:
    out = np.zeros(17)
    lib().or_rk4(C.byref(params), _dp(_d(s)), _dp(_d(u)), _dp(_d(dist)), float(h), _dp(out))
    return out


def project(params: Params, s) -> np.ndarray:
    s = _d(s).copy()
    lib().or_project(C.byref(params), _dp(s))
    return s


def action_to_rpm(params: Params, a: float) -> float:
    return lib().or_action_to_rpm(C.byref(params), float(a))


def stage(cfg: dict, t: int):
    w = Weights()
    sg = np.zeros(1)
    c = config(cfg)
    lib().or_stage(C.byref(c), int(t), C.byref(w), _dp(sg))
    return w, float(sg[0])


def reward(w: Weights, s, a) -> float:
    return lib().or_reward(C.byref(w), _dp(_d(s)), _dp(_d(a)))


def new_envs(n: int) -> np.ndarray:
    return np.zeros(n, dtype=ENV_DTYPE)


def reset(cfg: dict, env_id: int, counter: int) -> np.ndarray:
    e = new_envs(1)
    c = config(cfg)
    lib().or_reset(C.byref(c), int(env_id), int(counter), e.ctypes.data)
    return e[0]


def reset_many(cfg: dict, env_ids, counter: int) -> np.ndarray:
    env_ids = np.asarray(env_ids, dtype=np.uint64)
    e = new_envs(len(env_ids))
    c = config(cfg)
    L = lib()
    for i, eid in enumerate(env_ids):
        L.or_reset(C.byref(c), int(eid), int(counter), e[i:i + 1].ctypes.data)
    return e


def observe(cfg: dict, env: np.ndarray, env_id: int, t: int) -> np.ndarray:
    e = np.ascontiguousarray(np.asarray(env, dtype=ENV_DTYPE).reshape(1))
    obs = np.zeros(18 + 4 * int(cfg["n_hist"]))
    c = config(cfg)
    lib().or_observe(C.byref(c), e.ctypes.data, int(env_id), int(t), _dp(obs))
    return obs


def critic_observe(env: np.ndarray) -> np.ndarray:
    e = np.ascontiguousarray(np.asarray(env, dtype=ENV_DTYPE).reshape(1))
    obs = np.zeros(28)
    lib().or_critic_observe(e.ctypes.data, _dp(obs))
    return obs


def recompute_reward(cfg: dict, t: int, s1, a) -> float:
    c = config(cfg)
    return lib().or_recompute_reward(C.byref(c), int(t), _dp(_d(s1)), _dp(_d(a)))


class PolicyHandle:
    """Keeps the fp16 bit arrays alive behind an oracle Policy struct."""

    def __init__(self, w: dict):
        self.arrays = {k: np.ascontiguousarray(w[k], dtype=np.uint16) for k in
                       ("W1", "b1", "W2", "b2", "W3", "b3")}
        self.s = Policy()
        self.s.in_dim = int(self.arrays["W1"].shape[1])
        self.s.hidden = int(self.arrays["W1"].shape[0])
        for k, a in self.arrays.items():
            setattr(self.s, k, a.ctypes.data)


def mlp(policy: PolicyHandle, obs) -> np.ndarray:
    a = np.zeros(4)
    lib().or_mlp(C.byref(policy.s), _dp(_d(obs)), _dp(a))
    return a


def mlp_midpoint_margin(policy: PolicyHandle, obs) -> float:
    return lib().or_mlp_min_midpoint_margin(C.byref(policy.s), _dp(_d(obs)))


def env_step(cfg: dict, env: np.ndarray, env_id: int, t: int, a, stats=None):
    """One step of one env in place (env: a 1-element ENV_DTYPE array). Returns StepOut."""
    assert env.dtype == ENV_DTYPE and env.shape == (1,)
    so = StepOut()
    c = config(cfg)
    st = stats if stats is not None else np.zeros(len(STATS))
    lib().or_env_step(C.byref(c), env.ctypes.data, int(env_id), int(t), _dp(_d(a)), C.byref(so),
                      _dp(st))
    return so


def random_action(cfg: dict, env_id: int, t: int) -> np.ndarray:
    a = np.zeros(4)
    c = config(cfg)
    lib().or_random_action(C.byref(c), int(env_id), int(t), _dp(a))
    return a


def rollout(cfg: dict, envs: np.ndarray, env_ids, t0: int, T: int, mode: int,
            actions=None, policy: PolicyHandle | None = None, trace: bool = False,
            nthreads: int = 1):
    """Run T steps for every env (in place). actions: [T][n][4] for mode 0.
    Returns (stats[8], trace[T][n][28] or None)."""
    assert envs.dtype == ENV_DTYPE and envs.flags.c_contiguous
    n = len(envs)
    env_ids = np.ascontiguousarray(env_ids, dtype=np.uint64)
    assert env_ids.shape == (n,)
    act = None
    if mode == MODE_ACTIONS:
        act = _d(actions)
        assert act.shape == (T, n, 4)
    tr = np.zeros((T, n, TRACE_FIELDS)) if trace else None
    stats = np.zeros(len(STATS))
    c = config(cfg)
    lib().or_rollout(C.byref(c), envs.ctypes.data, env_ids.ctypes.data, n, int(t0), int(T),
                     int(mode), act.ctypes.data if act is not None else None,
                     C.byref(policy.s) if policy is not None else None,
                     tr.ctypes.data if tr is not None else None, _dp(stats), int(nthreads))
    return stats, tr


# ---- Lissajous tracking evaluation (f3) ------------------------------------------------
def lissajous(t: float, Tc: float, ax: float = 1.0, ay: float = 0.5, z: float = 0.0):
    """Reference position and velocity at time t (Q28)."""
    p, v = np.zeros(3), np.zeros(3)
    lib().or_lissajous(float(t), float(Tc), float(ax), float(ay), float(z), _dp(p), _dp(v))
    return p, v


def shift_observation(obs, p_ref, v_ref, clip_pos: float, clip_vel: float) -> np.ndarray:
    """Setpoint shifting with clipping (Q29) applied to an observation vector."""
    o = _d(obs).copy()
    lib().or_shift_observation(_dp(o), _dp(_d(p_ref)), _dp(_d(v_ref)), float(clip_pos), float(clip_vel))
    return o


def hover_rpm(params: Params) -> float:
    return lib().or_hover_rpm(C.byref(params))


def track(cfg: dict, policy: PolicyHandle | None, env_id: int, t0: int, Tc: float, n_steps: int,
          ax: float = 1.0, ay: float = 0.5, z: float = 0.0, clip_pos: float | None = None,
          clip_vel: float | None = None, trace: bool = False):
    """One env's Lissajous tracking run (Q28-Q31).  policy None = exact hover action.
    Returns (rmse, rmse_xy, steps_ok, positions[n_steps][3] or None)."""
    c = config(cfg)
    cp = cfg["init_pos"] if clip_pos is None else clip_pos
    cv = cfg["init_vel"] if clip_vel is None else clip_vel
    r, rxy = C.c_double(), C.c_double()
    ok = C.c_int32()
    tr = np.zeros((n_steps, 3)) if trace else None
    lib().or_track(C.byref(c), C.byref(policy.s) if policy is not None else None, int(env_id), int(t0),
                   float(Tc), float(ax), float(ay), float(z), float(cp), float(cv), int(n_steps),
                   C.byref(r), C.byref(rxy), C.byref(ok), tr.ctypes.data if tr is not None else None)
    return r.value, rxy.value, ok.value, tr


# ---- TD3 update (f4) ---------------------------------------------------------------------
TD3_DEFAULTS = {"gamma": 0.99, "tau": 0.005, "sigma_t": 0.2, "clip_t": 0.5, "lr_actor": 3e-4, "lr_critic": 3e-4,
                "beta1": 0.9, "beta2": 0.999, "eps": 1e-8}  # SPEC S:436 (the cited algorithm's defaults)


def net_size(n_in: int, hid: int, n_out: int) -> int:
    return int(lib().or_net_size(n_in, hid, n_out))


def td3_block_size(in_dim: int) -> int:
    na, nc = net_size(in_dim, 64, 4), net_size(32, 64, 1)
    return 2 * na + 4 * nc + 2 * na + 4 * nc


def td3_update(P: np.ndarray, in_dim: int, batch: dict, hyper: dict | None = None, t_critic: int = 1,
               t_actor: int = 1, update_actor: bool = True, want_grads: bool = False):
    """One TD3 update of one agent in place on the FP64 parameter block P (Q32-Q35).
    batch: o_a [B][I], o_c [B][28], a [B][4], r [B], o_a2, o_c2, done [B], eps [B][4].
    Returns (losses[3], grads or None)."""
    assert P.dtype == np.float64 and P.flags.c_contiguous and P.size == td3_block_size(in_dim)
    h = TD3Hyper(**{**TD3_DEFAULTS, **(hyper or {})})
    B = len(batch["r"])
    arr = {k: _d(batch[k]) for k in ("o_a", "o_c", "a", "r", "o_a2", "o_c2", "done", "eps")}
    losses = np.zeros(3)
    na, nc = net_size(in_dim, 64, 4), net_size(32, 64, 1)
    g = np.zeros(2 * nc + na) if want_grads else None
    lib().or_td3_update(_dp(P), int(in_dim), int(B), *(_dp(arr[k]) for k in
                                                       ("o_a", "o_c", "a", "r", "o_a2", "o_c2", "done", "eps")),
                        C.byref(h), int(t_critic), int(t_actor), int(bool(update_actor)), _dp(losses),
                        g.ctypes.data if g is not None else None)
    return losses, g
