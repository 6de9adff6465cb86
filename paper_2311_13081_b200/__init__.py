"""B200-native batched quadrotor environment of arXiv 2311.13081 ("Learning to Fly in Seconds").

Thin Python binding over the C ABI of ``libl2f.so`` (include/l2f.h).  Argument marshalling
only: every step of the method runs in the sm_100a kernels behind the ABI.  PyTorch provides
device memory (the env workspace and I/O tensors) and streams.  There is no CPU fallback:
importing this package without the built extension raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from .abi import (ABI_VERSION, DONE_DIVERGED, DONE_RESET, DONE_TERMINATED, DONE_TRUNCATED,  # noqa: F401
                  OBS_CORE, STATE_DIM, STATS, STATS_LEN, TRACE_FIELDS, L2FError, lib, make_config)

__all__ = ["Env", "Policy", "policy_forward", "TD3", "lib", "L2FError", "launch_count"]


def _stream(stream=None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _check(st: int, what: str):
    if st != 0:
        raise L2FError(f"{what}: status {st}: {lib().l2f_last_error().decode()}")


def launch_count() -> int:
    return int(lib().l2f_launch_count())


class Policy:
    """Actor MLP parameters as fp16 bit patterns (uint16 tensors), row-major [out][in]."""

    def __init__(self, weights: dict, device="cuda"):
        self.t = {k: torch.as_tensor(weights[k]).view(torch.int16).to(device).contiguous()
                  for k in ("W1", "b1", "W2", "b2", "W3", "b3")}
        self.in_dim = int(self.t["W1"].shape[1])
        self.hidden = int(self.t["W1"].shape[0])
        self.s = lib().make_policy(*(self.t[k].data_ptr() for k in ("W1", "b1", "W2", "b2", "W3", "b3")),
                                   self.in_dim, self.hidden)


class HostPolicy:
    """Same, in pinned host memory (for l2f_rollout_host)."""

    def __init__(self, weights: dict):
        self.t = {k: torch.as_tensor(weights[k]).view(torch.int16).contiguous().pin_memory()
                  for k in ("W1", "b1", "W2", "b2", "W3", "b3")}
        self.in_dim = int(self.t["W1"].shape[1])
        self.hidden = int(self.t["W1"].shape[0])
        self.s = lib().make_policy(*(self.t[k].data_ptr() for k in ("W1", "b1", "W2", "b2", "W3", "b3")),
                                   self.in_dim, self.hidden)


def policy_forward(policy: Policy, obs: torch.Tensor, stream=None) -> torch.Tensor:
    """obs [n][in_dim] fp32 (cuda) -> tanh actions [n][4] (before exploration noise)."""
    assert obs.is_cuda and obs.dtype == torch.float32 and obs.is_contiguous()
    out = torch.empty(obs.shape[0], 4, device=obs.device, dtype=torch.float32)
    _check(lib().l2f_policy_forward(C.byref(policy.s), _ptr(obs), _ptr(out), obs.shape[0], _stream(stream)),
           "l2f_policy_forward")
    return out


class Env:
    """N independent quadrotor environments resident in HBM (one workspace tensor)."""

    def __init__(self, cfg: dict, num_envs: int, env_id_offset: int = 0, device="cuda"):
        L = lib()
        self.cfg_dict = cfg
        self.n = int(num_envs)
        self.n_hist = int(cfg["n_hist"])
        self.device = torch.device(device)
        self.cfg = make_config(cfg, self.n, env_id_offset)
        nbytes = C.c_size_t()
        _check(L.l2f_workspace_size(C.byref(self.cfg), C.byref(nbytes)), "l2f_workspace_size")
        self.ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.device)
        self.h = C.c_void_p()
        _check(L.l2f_create(C.byref(self.cfg), _ptr(self.ws), nbytes, C.byref(self.h)), "l2f_create")
        self._views()

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().l2f_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _views(self):
        v = lib().StateView()
        _check(lib().l2f_get_state(self.h, C.byref(v)), "l2f_get_state")
        base = self.ws.data_ptr()
        n, nh = self.n, max(self.n_hist, 1)

        def view(ptr, count, dtype, shape):
            off = int(ptr) - base
            esz = torch.empty(0, dtype=dtype).element_size()
            return self.ws[off: off + count * esz].view(dtype).view(*shape)

        # raw workspace views in the ABI layout (include/l2f.h): float4 groups + a tail block
        self._grp = {}
        for name, ptr, c in (("state", v.state, 17), ("dist", v.dist, 6), ("dr", v.dr, 5)):
            self._grp[name] = (view(ptr, c * n, torch.float32, (c * n,)), c)
        self.hist4 = view(v.hist, nh * 4 * n, torch.float32, (nh, n, 4))
        self.hist_t0 = view(v.hist_t0, n, torch.int32, (n,))
        self.hist_fill4 = view(v.hist_fill, 4 * n, torch.float32, (n, 4))
        self.ep_step = view(v.ep_step, n, torch.int32, (n,))
        self.ep_return = view(v.ep_return, n, torch.float32, (n,))

    def _g2l(self, name) -> torch.Tensor:  # raw grouped array -> [C][N] (copy)
        flat, c = self._grp[name]
        n, g, r = self.n, c // 4, c % 4
        parts = [flat[:4 * g * n].view(g, n, 4).permute(0, 2, 1).reshape(4 * g, n)]
        if r:
            parts.append(flat[4 * g * n:].view(n, r).t())
        return torch.cat(parts, 0).contiguous()

    def raw(self, name) -> torch.Tensor:
        """The flat workspace view of a grouped array (state / dist / dr), ABI layout."""
        return self._grp[name][0]

    @property
    def state(self) -> torch.Tensor:
        """[17][N] copy of the state (component-major)."""
        return self._g2l("state")

    @property
    def dist(self) -> torch.Tensor:
        return self._g2l("dist")

    @property
    def dr(self) -> torch.Tensor:
        return self._g2l("dr")

    @property
    def hist(self) -> torch.Tensor:
        """[N_H][4][N] copy of the action-history ring."""
        return self.hist4.permute(0, 2, 1).contiguous()

    @property
    def hist_fill(self) -> torch.Tensor:
        """[4][N] copy of the episodes' history fill values."""
        return self.hist_fill4.t().contiguous()

    def set_logical(self, name: str, value):
        """Write a component-major array (as returned by the properties above) into the workspace."""
        x = torch.as_tensor(value).to(device=self.device)
        if name in self._grp:
            flat, c = self._grp[name]
            n, g, r = self.n, c // 4, c % 4
            x = x.to(torch.float32)
            flat[:4 * g * n].view(g, n, 4).copy_(x[:4 * g].reshape(g, 4, n).permute(0, 2, 1))
            if r:
                flat[4 * g * n:].view(n, r).copy_(x[4 * g:].t())
        elif name == "hist":
            self.hist4.copy_(x.to(torch.float32).permute(0, 2, 1))
        elif name == "hist_fill":
            self.hist_fill4.copy_(x.to(torch.float32).t())
        else:
            getattr(self, name).copy_(x)

    # -------------------------------------------------------------------------------
    @property
    def t(self) -> int:
        v = lib().StateView()
        _check(lib().l2f_get_state(self.h, C.byref(v)), "l2f_get_state")
        return int(v.t)

    @t.setter
    def t(self, value: int):
        _check(lib().l2f_set_t(self.h, int(value)), "l2f_set_t")

    def get_state(self) -> dict:
        """Copy of the full env state (device tensors, the raw ABI layouts) for checkpointing;
        see set_state."""
        return {"state": self.raw("state").clone(), "dist": self.raw("dist").clone(), "dr": self.raw("dr").clone(),
                "hist": self.hist4.clone(), "hist_t0": self.hist_t0.clone(), "hist_fill": self.hist_fill4.clone(),
                "ep_step": self.ep_step.clone(), "ep_return": self.ep_return.clone(), "t": self.t}

    def set_state(self, snap: dict, stream=None):
        """l2f_set_state: restore (a subset of) a get_state() snapshot; missing keys stay."""
        v = lib().StateView()
        keep = []

        def ptr(name, dtype):
            x = snap.get(name)
            if x is None:
                return None
            x = x.to(device=self.device, dtype=dtype).contiguous()
            keep.append(x)
            return C.c_void_p(x.data_ptr())

        v.state = ptr("state", torch.float32)
        v.dist = ptr("dist", torch.float32)
        v.dr = ptr("dr", torch.float32)
        v.hist = ptr("hist", torch.float32)
        v.hist_t0 = ptr("hist_t0", torch.int32)
        v.hist_fill = ptr("hist_fill", torch.float32)
        v.ep_step = ptr("ep_step", torch.int32)
        v.ep_return = ptr("ep_return", torch.float32)
        v.t = int(snap.get("t", self.t))
        # sizes as the snapshot has them (the library rejects a mismatch before copying)
        per_env = {"state": 17, "dist": 6, "dr": 5}  # flat raw arrays: C x N floats
        ns = set()
        for k in ("state", "dist", "dr", "hist", "hist_fill", "hist_t0", "ep_step", "ep_return"):
            x = snap.get(k)
            if x is None:
                continue
            ns.add(int(x.numel() // per_env[k]) if k in per_env else int(x.shape[1] if k == "hist" else x.shape[0]))
        if len(ns) > 1:
            raise L2FError(f"set_state: inconsistent env counts {sorted(ns)}")
        v.num_envs = ns.pop() if ns else self.n
        h = snap.get("hist")
        v.action_history = (int(h.shape[0]) if self.n_hist > 0 else 0) if h is not None else self.n_hist
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(lib().l2f_set_state(self.h, C.byref(v), C.c_void_p(s.cuda_stream)), "l2f_set_state")
        s.synchronize()  # the source tensors in `keep` must outlive the copies

    def make_out(self, obs_core=True, reward=True, flags=True, final_state=False, obs_dense=False,
                 obs_critic=False):
        d = self.device
        return {
            "obs_critic": torch.empty(28, self.n, device=d) if obs_critic else None,
            "obs_core": torch.empty(18, self.n, device=d) if obs_core else None,
            "reward": torch.empty(self.n, device=d) if reward else None,
            "flags": torch.empty(self.n, device=d, dtype=torch.uint8) if flags else None,
            "final_state": torch.empty(17, self.n, device=d) if final_state else None,
            "obs_dense": torch.empty(self.n, 18 + 4 * self.n_hist, device=d) if obs_dense else None,
        }

    def _out_struct(self, out: dict | None):
        if out is None:
            return None
        o = lib().StepOut()
        for k in ("obs_core", "obs_dense", "reward", "flags", "final_state", "obs_critic"):
            t = out.get(k)
            if t is not None:
                assert t.is_cuda and t.is_contiguous()
                setattr(o, k, t.data_ptr())
        return C.byref(o)

    def reset(self, mask: torch.Tensor | None = None, out: dict | None = None, stream=None):
        if mask is not None:
            assert mask.dtype == torch.uint8 and mask.is_cuda and mask.numel() == self.n
        _check(lib().l2f_reset(self.h, _ptr(mask), self._out_struct(out), _stream(stream)), "l2f_reset")
        return out

    def step(self, actions: torch.Tensor, out: dict | None = None, stream=None):
        assert actions.is_cuda and actions.dtype == torch.float32 and actions.is_contiguous()
        assert actions.shape == (4, self.n)
        _check(lib().l2f_step(self.h, _ptr(actions), self._out_struct(out), _stream(stream)), "l2f_step")
        return out

    def rollout(self, T: int, policy: Policy | None = None, actions: torch.Tensor | None = None,
                trace_ids: torch.Tensor | None = None, stream=None):
        trace = None
        K = 0
        if actions is not None:
            assert actions.is_cuda and actions.dtype == torch.float32 and actions.shape == (T, 4, self.n)
            actions = actions.contiguous()
        if trace_ids is not None:
            trace_ids = trace_ids.to(device=self.device, dtype=torch.int64).contiguous()
            K = int(trace_ids.numel())
            trace = torch.zeros(T, K, TRACE_FIELDS, device=self.device)
        self._keep = (actions, trace_ids)  # (alive while the asynchronous launch reads them)
        _check(lib().l2f_rollout(self.h, C.byref(policy.s) if policy is not None else None, _ptr(actions), int(T),
                                 _ptr(trace), _ptr(trace_ids), K, _stream(stream)), "l2f_rollout")
        return trace

    def track(self, policy: Policy, cycle_time, n_steps: int, amp_x: float = 1.0, amp_y: float = 0.5,
              altitude: float = 0.0, clip_pos: float | None = None, clip_vel: float | None = None, stream=None):
        """l2f_track: batched Lissajous tracking with setpoint shifting (f3).  cycle_time: a
        float or a [N] tensor of per-env cycle times (s).  Clip bounds default to the training
        initial-state bounds (init_pos, init_vel).  Returns {rmse, rmse_xy, steps_ok} ([N])."""
        from .abi import Tracking
        d = self.device
        ct = torch.as_tensor(cycle_time, dtype=torch.float32, device=d)
        if ct.dim() == 0:
            ct = ct.expand(self.n)
        ct = ct.contiguous()
        assert ct.shape == (self.n,)
        out = {"rmse": torch.empty(self.n, device=d), "rmse_xy": torch.empty(self.n, device=d),
               "steps_ok": torch.empty(self.n, dtype=torch.int32, device=d)}
        sp = Tracking()
        sp.cycle_time = ct.data_ptr()
        sp.amp_x, sp.amp_y, sp.altitude = float(amp_x), float(amp_y), float(altitude)
        sp.clip_pos = float(self.cfg.init_pos if clip_pos is None else clip_pos)
        sp.clip_vel = float(self.cfg.init_vel if clip_vel is None else clip_vel)
        sp.n_steps = int(n_steps)
        sp.rmse, sp.rmse_xy, sp.steps_ok = (out[k].data_ptr() for k in ("rmse", "rmse_xy", "steps_ok"))
        self._keep = ct  # (alive while the asynchronous launch reads it)
        _check(lib().l2f_track(self.h, C.byref(policy.s), C.byref(sp), _stream(stream)), "l2f_track")
        return out

    def recompute_rewards(self, t: int, next_state: torch.Tensor, actions: torch.Tensor, stream=None):
        """Rewards of stored transitions (s' [17][M], a' [4][M]) under the curriculum stage of
        step t (P:231 reward recalculation)."""
        assert next_state.is_cuda and actions.is_cuda and next_state.shape[0] == 17 and actions.shape[0] == 4
        m = next_state.shape[1]
        assert actions.shape[1] == m and next_state.is_contiguous() and actions.is_contiguous()
        out = torch.empty(m, device=next_state.device)
        _check(lib().l2f_recompute_rewards(self.h, int(t), _ptr(next_state), _ptr(actions), m, _ptr(out),
                                           _stream(stream)), "l2f_recompute_rewards")
        return out

    def episode_stats(self, reset: bool = False, stream=None) -> torch.Tensor:
        out = torch.empty(STATS_LEN, dtype=torch.float64, device=self.device)
        _check(lib().l2f_episode_stats(self.h, _ptr(out), int(reset), _stream(stream)), "l2f_episode_stats")
        return out

    # host-buffer entry points (synchronous) ----------------------------------------
    def step_host(self, h_actions: torch.Tensor, h_obs=None, h_reward=None, h_flags=None, stream=None):
        assert not h_actions.is_cuda and h_actions.dtype == torch.float32 and h_actions.is_contiguous()
        _check(lib().l2f_step_host(self.h, _ptr(h_actions), _ptr(h_obs), _ptr(h_reward), _ptr(h_flags),
                                   _stream(stream)), "l2f_step_host")

    def rollout_host(self, policy: HostPolicy, T: int, h_stats: torch.Tensor | None = None, reset_stats=True,
                     stream=None):
        if h_stats is not None:
            assert h_stats.dtype == torch.float64 and not h_stats.is_cuda
        _check(lib().l2f_rollout_host(self.h, C.byref(policy.s), int(T), _ptr(h_stats), int(reset_stats),
                                      _stream(stream)), "l2f_rollout_host")
        return h_stats


class TD3:
    """Batched TD3 learner of n_agents independent agents (l2f_td3_update).
    params [A][block] FP32: [actor, actor', Q1, Q2, Q1', Q2', m/v of actor, Q1, Q2] (include/l2f.h)."""

    DEFAULTS = {"gamma": 0.99, "tau": 0.005, "sigma_t": 0.2, "clip_t": 0.5, "lr_actor": 3e-4, "lr_critic": 3e-4,
                "beta1": 0.9, "beta2": 0.999, "eps": 1e-8}

    def __init__(self, n_agents: int, in_dim: int, batch: int = 256, hyper: dict | None = None, device="cuda"):
        from .abi import TD3Hyper
        blk, sb = C.c_int64(), C.c_int64()
        _check(lib().l2f_td3_sizes(int(in_dim), int(batch), C.byref(blk), C.byref(sb)), "l2f_td3_sizes")
        self.A, self.in_dim, self.B, self.device = int(n_agents), int(in_dim), int(batch), device
        self.block, self.scratch_bytes = int(blk.value), int(sb.value)
        self.params = torch.zeros(self.A, self.block, device=device)
        self.scratch = torch.zeros(self.A * self.scratch_bytes, dtype=torch.uint8, device=device)
        self.losses = torch.zeros(self.A, 3, device=device)
        self.hyper = {**self.DEFAULTS, **(hyper or {})}
        self.h = TD3Hyper(**self.hyper)
        self.t_critic = self.t_actor = 0
        self.na = 64 * in_dim + 64 + 64 * 64 + 64 + 4 * 64 + 4
        self.nc = 64 * 32 + 64 + 64 * 64 + 64 + 64 + 1

    def offsets(self) -> dict:
        na, nc = self.na, self.nc
        o = {"actor": 0, "actor_t": na, "q1": 2 * na, "q2": 2 * na + nc, "q1_t": 2 * na + 2 * nc,
             "q2_t": 2 * na + 3 * nc, "m_actor": 2 * na + 4 * nc, "v_actor": 3 * na + 4 * nc,
             "m_q1": 4 * na + 4 * nc, "v_q1": 4 * na + 5 * nc, "m_q2": 4 * na + 6 * nc, "v_q2": 4 * na + 7 * nc}
        return o

    def update(self, batch: dict, update_actor: bool, stream=None):
        """One update of every agent; batch tensors [A][B][...] fp32 on the device."""
        from .abi import TD3Batch
        A, B, I = self.A, self.B, self.in_dim
        shapes = {"o_a": (A, B, I), "o_c": (A, B, 28), "a": (A, B, 4), "r": (A, B), "o_a2": (A, B, I),
                  "o_c2": (A, B, 28), "done": (A, B), "eps": (A, B, 4)}
        for k, shp in shapes.items():
            if tuple(batch[k].shape) != shp:
                raise ValueError(f"TD3 batch[{k!r}] has shape {tuple(batch[k].shape)}, expected {shp}")
        keep = {k: batch[k].to(device=self.device, dtype=torch.float32).contiguous() for k in shapes}
        self._keep = keep  # (converted copies stay alive while the asynchronous update reads them)
        b = TD3Batch(**{k: v.data_ptr() for k, v in keep.items()})
        self.t_critic += 1
        if update_actor:
            self.t_actor += 1
        _check(lib().l2f_td3_update(_ptr(self.params), self.A, self.in_dim, self.B, C.byref(b), C.byref(self.h),
                                    self.t_critic, max(self.t_actor, 1), int(bool(update_actor)), _ptr(self.losses),
                                    _ptr(self.scratch), _stream(stream)), "l2f_td3_update")
        return self.losses

    def grads(self) -> dict:
        """Raw gradients of the last update (per agent views into the scratch): q1, q2, actor."""
        f = self.scratch.view(torch.float32).view(self.A, self.scratch_bytes // 4)
        g0 = self.B * (1 + 32 + 4 * 64 + 1 + 2 * 64 + 4 + 2 * 64 + 4)
        return {"q1": f[:, g0:g0 + self.nc], "q2": f[:, g0 + self.nc:g0 + 2 * self.nc],
                "actor": f[:, g0 + 2 * self.nc:g0 + 2 * self.nc + self.na]}

    def actor_policy(self, agent: int = 0, stream=None) -> "Policy":
        """The agent's actor as a device fp16 Policy (l2f_td3_export_actor; no host round trip)."""
        from .abi import PolicyS
        pol = Policy.__new__(Policy)
        buf = torch.empty(self.na, dtype=torch.int16, device=self.device)
        pol.t = {"buf": buf}
        pol.in_dim, pol.hidden = self.in_dim, 64
        pol.s = PolicyS()
        _check(lib().l2f_td3_export_actor(_ptr(self.params), int(agent), self.in_dim, _ptr(buf), C.byref(pol.s),
                                          _stream(stream)), "l2f_td3_export_actor")
        return pol

    def actor_policy_weights(self, agent: int = 0) -> dict:
        """The agent's actor as fp16 bit patterns in the l2f_policy layout (for Policy / rollouts)."""
        import numpy as np
        p = self.params[agent, :self.na].cpu().numpy()
        I, o = self.in_dim, 0
        out = {}
        for k, n in (("W1", 64 * I), ("b1", 64), ("W2", 64 * 64), ("b2", 64), ("W3", 4 * 64), ("b3", 4)):
            a = p[o:o + n].astype(np.float16).view(np.uint16)
            out[k] = a.reshape(64, I) if k == "W1" else (a.reshape(64, 64) if k == "W2" else
                                                          (a.reshape(4, 64) if k == "W3" else a))
            o += n
        return out
