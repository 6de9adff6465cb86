"""GPU <-> oracle parity of the batched Lissajous tracking evaluation, l2f_track (SURVEY 8(f)
f3; P:154 setpoint shifting + clipping, P:305-306 reference, Table III RMSE; Q28-Q31).

A zero-weight actor is deterministic and symmetric (no chaos), so its tracking RMSE and
failure step are compared with the oracle tightly; a random hover-biased actor is compared
over a short horizon, where the closed-loop fp16/fp32 vs FP64 trajectories still agree."""
import math

import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2311_13081_b200 as p
    p.lib()
    return p


def zero_policy(in_dim=146, bias=0.0):
    z = lambda *s: np.zeros(s, dtype=np.float16).view(np.uint16)  # noqa: E731
    b3 = np.full(4, bias, dtype=np.float16).view(np.uint16)
    return {"W1": z(64, in_dim), "b1": z(64), "W2": z(64, 64), "b2": z(64), "W3": z(4, 64), "b3": b3}


def cycle_times(n):
    return np.array([(15.0, 5.5, 3.5)[i % 3] for i in range(n)], dtype=np.float32)


@pytest.mark.parametrize("terminate", [True, False])
def test_track_zero_actor_matches_oracle(pkg, terminate):
    """a = 0 for every env: the vehicle climbs straight up from p_ref(0) while the reference
    moves; RMSE (3-D and x-y) and the failure step vs the oracle, per cycle time."""
    cfg = inputs.config_c4()
    if not terminate:
        cfg["flags"] &= ~4
    n, steps = 3 * 128 + 31, 400
    W = zero_policy()
    env = pkg.Env(cfg, n)
    env.reset()
    T = cycle_times(n)
    out = env.track(pkg.Policy(W), torch.as_tensor(T, device="cuda"), steps, altitude=0.5)
    r, rxy, ok = (out[k].cpu().numpy() for k in ("rmse", "rmse_xy", "steps_ok"))
    ph = oracle.PolicyHandle(W)
    for i in list(range(6)) + [n - 1]:
        orr, orxy, ook, _ = oracle.track(cfg, ph, i, 0, float(T[i]), steps, z=0.5)
        assert ok[i] == ook, (i, ok[i], ook)
        assert abs(r[i] - orr) <= 1e-5 + 1e-4 * orr, (i, r[i], orr)
        assert abs(rxy[i] - orxy) <= 1e-5 + 1e-4 * orxy, (i, rxy[i], orxy)
    # identical actors and cycle times give identical results (no RNG in this path)
    for j in range(3):
        assert np.all(r[j::3] == r[j]) and np.all(ok[j::3] == ok[j])
    if terminate:
        assert (ok < steps).all()  # climbing away fails eventually
    else:
        assert (ok == steps).all()
    assert env.t == steps


def test_track_random_actor_short_horizon_matches_oracle(pkg):
    """Hover-biased random actor with observation noise (C4), 60 steps (0.6 s) of closed-loop
    tracking: RMSE within 2e-3 m + 2 % of the oracle's; the same success flags."""
    cfg = inputs.config_c4()
    n, steps = 3 * 128, 60
    W = inputs.policy_weights(146, 64, seed=5, out_bias=inputs.hover_policy_bias())
    env = pkg.Env(cfg, n)
    env.reset()
    env.t = 1000
    T = cycle_times(n)
    out = env.track(pkg.Policy(W), torch.as_tensor(T, device="cuda"), steps)
    r, rxy, ok = (out[k].cpu().numpy() for k in ("rmse", "rmse_xy", "steps_ok"))
    ph = oracle.PolicyHandle(W)
    for i in range(0, n, 19):
        orr, orxy, ook, _ = oracle.track(cfg, ph, i, 1000, float(T[i]), steps)
        assert (ok[i] == steps) == (ook == steps), (i, ok[i], ook)
        m = min(ok[i], ook)
        if m == steps:
            assert abs(r[i] - orr) <= 2e-3 + 0.02 * orr, (i, r[i], orr)
            assert abs(rxy[i] - orxy) <= 2e-3 + 0.02 * orxy, (i, rxy[i], orxy)
    assert np.isfinite(r).all() and (r >= rxy - 1e-6).all()
    assert env.t == 1000 + steps


def test_track_leaves_a_consistent_env(pkg):
    """After l2f_track the env holds the final tracking state with a valid history ring, so
    rollouts continue from it (and l2f_reset restores training)."""
    cfg = inputs.config_c4()
    n = 256
    W = inputs.policy_weights(146, 64, seed=5, out_bias=inputs.hover_policy_bias())
    pol = pkg.Policy(W)
    env = pkg.Env(cfg, n)
    env.reset()
    env.track(pol, 5.5, 50)
    assert int(env.hist_t0[0]) == 50 - cfg["n_hist"]
    assert torch.isfinite(env.state).all()
    env.rollout(10, policy=pol)
    env.reset()
    assert torch.isfinite(env.state).all()


def test_track_invalid_arguments(pkg):
    cfg = inputs.config_c4()
    env = pkg.Env(cfg, 128)
    pol = pkg.Policy(inputs.policy_weights(146, 64))
    with pytest.raises(Exception):
        env.track(pol, 5.5, 0)
    with pytest.raises(Exception):
        env.track(pol, 5.5, 10, clip_pos=0.0)
    bad = pkg.Policy(inputs.policy_weights(18 + 16, 64))
    with pytest.raises(Exception):
        env.track(bad, 5.5, 10)


@pytest.mark.parametrize("n,steps", [(1, 1), (129, 3)])
def test_track_tiny_runs_match_oracle(pkg, n, steps):
    cfg = inputs.config_c4()
    W = inputs.policy_weights(146, 64, seed=5, out_bias=inputs.hover_policy_bias())
    env = pkg.Env(cfg, n)
    env.reset()
    out = env.track(pkg.Policy(W), 5.5, steps)
    r, ok = out["rmse"].cpu().numpy(), out["steps_ok"].cpu().numpy()
    ph = oracle.PolicyHandle(W)
    for i in (0, n - 1):
        orr, _, ook, _ = oracle.track(cfg, ph, i, 0, 5.5, steps)
        assert ok[i] == ook and abs(r[i] - orr) <= 1e-4 + 1e-3 * orr


def test_track_full_size_sampled(pkg):
    """The bench's tracking configuration (2^20 envs, Table III cycle times), sampled envs vs
    the oracle with the deterministic zero actor (no chaos: tight agreement)."""
    cfg = inputs.config_c4()
    n, steps = 1 << 20, 120
    W = zero_policy()
    env = pkg.Env(cfg, n)
    T = cycle_times(n)
    out = env.track(pkg.Policy(W), torch.as_tensor(T, device="cuda"), steps)
    r, ok = out["rmse"].cpu().numpy(), out["steps_ok"].cpu().numpy()
    ph = oracle.PolicyHandle(W)
    for i in inputs.trace_ids(n, 12, seed=9):
        orr, _, ook, _ = oracle.track(cfg, ph, int(i), 0, float(T[i]), steps)
        assert ok[i] == ook and abs(r[i] - orr) <= 1e-5 + 1e-4 * orr, (i, r[i], orr, ok[i], ook)
