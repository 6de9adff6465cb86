"""ctypes mirror of include/l2f.h and config marshalling (dict -> l2f_config)."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# L2F_LIB_PATH: another build of the same library (e.g. the -DL2F_DEBUG_CHECKS build of
# scripts/debug_checks.sh); default the in-tree libl2f.so
LIB_PATH = os.environ.get("L2F_LIB_PATH") or os.path.join(HERE, "libl2f.so")

ABI_VERSION = 2
STATE_DIM, OBS_CORE, MAX_HIST, STATS_LEN, TRACE_FIELDS = 17, 18, 32, 8, 32
DONE_TERMINATED, DONE_TRUNCATED, DONE_DIVERGED, DONE_RESET = 1, 2, 4, 8
STATS = ["episodes", "terminated", "truncated", "diverged", "sum_len", "sum_ret", "sum_ret_sq", "env_steps"]
EXPORTS = ["l2f_workspace_size", "l2f_create", "l2f_destroy", "l2f_reset", "l2f_step", "l2f_rollout",
           "l2f_episode_stats", "l2f_step_host", "l2f_rollout_host", "l2f_get_state", "l2f_set_t", "l2f_set_state", "l2f_track", "l2f_td3_sizes", "l2f_td3_update", "l2f_td3_export_actor",
           "l2f_policy_forward", "l2f_recompute_rewards", "l2f_selftest_philox", "l2f_launch_count", "l2f_last_error", "l2f_abi_version"]


class L2FError(RuntimeError):
    pass


class Params(C.Structure):
    _fields_ = [("mass", C.c_double), ("J", C.c_double * 3), ("rotor_pos", (C.c_double * 3) * 4),
                ("spin_dir", C.c_double * 4), ("thrust_c", C.c_double * 3), ("torque_c", C.c_double),
                ("motor_tau", C.c_double), ("rpm_min", C.c_double), ("rpm_max", C.c_double),
                ("gravity", C.c_double)]


class RewardWeights(C.Structure):
    _fields_ = [("C_rp", C.c_double), ("C_rq", C.c_double), ("C_rv", C.c_double), ("C_rw", C.c_double),
                ("C_ra", C.c_double), ("C_rab", C.c_double * 4), ("C_rs", C.c_double)]


class Curriculum(C.Structure):
    _fields_ = [("init", RewardWeights), ("target", RewardWeights), ("factor", RewardWeights),
                ("sigma_init", C.c_double), ("sigma_target", C.c_double), ("sigma_factor", C.c_double),
                ("interval", C.c_int64)]


class Config(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("flags", C.c_uint32), ("num_envs", C.c_int64),
                ("env_id_offset", C.c_uint64), ("seed", C.c_uint64), ("action_history", C.c_int32),
                ("max_episode_steps", C.c_int32), ("dt", C.c_double), ("params", Params),
                ("dr_lo", C.c_double), ("dr_hi", C.c_double), ("init_pos", C.c_double),
                ("init_angle", C.c_double), ("init_vel", C.c_double), ("init_angvel", C.c_double),
                ("init_rpm_lo", C.c_double), ("init_rpm_hi", C.c_double), ("dist_force", C.c_double),
                ("dist_torque", C.c_double), ("obs_sigma", C.c_double * 4), ("term_pos", C.c_double),
                ("term_vel", C.c_double), ("term_angvel", C.c_double), ("curriculum", Curriculum)]


class StepOut(C.Structure):
    _fields_ = [("obs_core", C.c_void_p), ("obs_dense", C.c_void_p), ("reward", C.c_void_p),
                ("flags", C.c_void_p), ("final_state", C.c_void_p), ("obs_critic", C.c_void_p)]


class PolicyS(C.Structure):
    _fields_ = [("W1", C.c_void_p), ("b1", C.c_void_p), ("W2", C.c_void_p), ("b2", C.c_void_p),
                ("W3", C.c_void_p), ("b3", C.c_void_p), ("in_dim", C.c_int32), ("hidden", C.c_int32)]


class Tracking(C.Structure):
    _fields_ = [("cycle_time", C.c_void_p), ("amp_x", C.c_double), ("amp_y", C.c_double),
                ("altitude", C.c_double), ("clip_pos", C.c_double), ("clip_vel", C.c_double),
                ("n_steps", C.c_int32), ("rmse", C.c_void_p), ("rmse_xy", C.c_void_p), ("steps_ok", C.c_void_p)]


class TD3Hyper(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("gamma", "tau", "sigma_t", "clip_t", "lr_actor", "lr_critic", "beta1",
                                          "beta2", "eps")]


class TD3Batch(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("o_a", "o_c", "a", "r", "o_a2", "o_c2", "done", "eps")]


class StateView(C.Structure):
    _fields_ = [("state", C.c_void_p), ("dist", C.c_void_p), ("dr", C.c_void_p), ("hist", C.c_void_p),
                ("hist_t0", C.c_void_p), ("hist_fill", C.c_void_p), ("ep_step", C.c_void_p), ("ep_return", C.c_void_p), ("t", C.c_uint64),
                ("num_envs", C.c_int64), ("action_history", C.c_int32)]


def _weights(d) -> RewardWeights:
    w = RewardWeights()
    for k in ("C_rp", "C_rq", "C_rv", "C_rw", "C_ra", "C_rs"):
        setattr(w, k, float(d[k]))
    for i in range(4):
        w.C_rab[i] = float(d["C_rab"][i])
    return w


def make_config(d: dict, num_envs: int, env_id_offset: int = 0) -> Config:
    c = Config()
    c.abi_version = ABI_VERSION
    c.flags = int(d["flags"])
    c.num_envs = int(num_envs)
    c.env_id_offset = int(env_id_offset)
    c.seed = int(d["seed"])
    c.action_history = int(d["n_hist"])
    c.max_episode_steps = int(d["max_episode_steps"])
    c.dt = float(d["dt"])
    p = d["params"]
    c.params.mass = p["mass"]
    for i in range(3):
        c.params.J[i] = p["J"][i]
        c.params.thrust_c[i] = p["thrust_c"][i]
    for i in range(4):
        for j in range(3):
            c.params.rotor_pos[i][j] = p["rotor_pos"][i][j]
        c.params.spin_dir[i] = p["spin_dir"][i]
    c.params.torque_c = p["torque_c"]
    c.params.motor_tau = p["motor_tau"]
    c.params.rpm_min = p["rpm_min"]
    c.params.rpm_max = p["rpm_max"]
    c.params.gravity = p["gravity"]
    c.dr_lo, c.dr_hi = d["dr_range"]
    c.init_pos, c.init_angle, c.init_vel, c.init_angvel = d["init_pos"], d["init_angle"], d["init_vel"], d["init_angvel"]
    c.init_rpm_lo, c.init_rpm_hi = d["init_rpm"]
    c.dist_force, c.dist_torque = d["dist_force"], d["dist_torque"]
    for i in range(4):
        c.obs_sigma[i] = d["obs_sigma"][i]
    c.term_pos, c.term_vel, c.term_angvel = d["term_pos"], d["term_vel"], d["term_angvel"]
    cur = d["curriculum"]
    c.curriculum.init = _weights(cur["init"])
    c.curriculum.target = _weights(cur["target"])
    c.curriculum.factor = _weights(cur["factor"])
    c.curriculum.sigma_init = cur["sigma_init"]
    c.curriculum.sigma_target = cur["sigma_target"]
    c.curriculum.sigma_factor = cur["sigma_factor"]
    c.curriculum.interval = int(cur["interval"])
    return c


_lib = None


def lib():
    """Load libl2f.so (built in-tree by __graft_entry__.build()).  Fails loudly if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise L2FError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, st = C.c_void_p, C.c_int
        L.l2f_workspace_size.argtypes = [C.POINTER(Config), C.POINTER(C.c_size_t)]
        L.l2f_create.argtypes = [C.POINTER(Config), vp, C.c_size_t, C.POINTER(vp)]
        L.l2f_destroy.argtypes = [vp]
        L.l2f_reset.argtypes = [vp, vp, C.POINTER(StepOut), vp]
        L.l2f_step.argtypes = [vp, vp, C.POINTER(StepOut), vp]
        L.l2f_rollout.argtypes = [vp, C.POINTER(PolicyS), vp, C.c_int32, vp, vp, C.c_int32, vp]
        L.l2f_episode_stats.argtypes = [vp, vp, C.c_int32, vp]
        L.l2f_step_host.argtypes = [vp, vp, vp, vp, vp, vp]
        L.l2f_rollout_host.argtypes = [vp, C.POINTER(PolicyS), C.c_int32, vp, C.c_int32, vp]
        L.l2f_get_state.argtypes = [vp, C.POINTER(StateView)]
        L.l2f_set_t.argtypes = [vp, C.c_uint64]
        L.l2f_set_state.argtypes = [vp, C.POINTER(StateView), vp]
        L.l2f_track.argtypes = [vp, vp, C.POINTER(Tracking), vp]
        L.l2f_td3_sizes.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.l2f_td3_export_actor.argtypes = [vp, C.c_int32, C.c_int32, vp, C.POINTER(PolicyS), vp]
        L.l2f_td3_update.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.POINTER(TD3Batch), C.POINTER(TD3Hyper),
                                     C.c_int64, C.c_int64, C.c_int32, vp, vp, vp]
        L.l2f_policy_forward.argtypes = [C.POINTER(PolicyS), vp, vp, C.c_int64, vp]
        L.l2f_recompute_rewards.argtypes = [vp, C.c_uint64, vp, vp, C.c_int64, vp, vp]
        L.l2f_selftest_philox.argtypes = [C.c_int64, C.c_uint64, C.c_uint32, vp, vp, vp]
        L.l2f_launch_count.restype = C.c_uint64
        L.l2f_launch_count.argtypes = []
        L.l2f_last_error.restype = C.c_char_p
        L.l2f_abi_version.restype = C.c_int32
        for f in EXPORTS:
            if f not in ("l2f_launch_count", "l2f_last_error", "l2f_abi_version"):
                getattr(L, f).restype = st
        if L.l2f_abi_version() != ABI_VERSION:
            raise L2FError("libl2f.so ABI version mismatch")
        L.StepOut = StepOut
        L.StateView = StateView
        L.make_policy = lambda W1, b1, W2, b2, W3, b3, i, h: PolicyS(W1, b1, W2, b2, W3, b3, i, h)
        _lib = L
    return _lib
