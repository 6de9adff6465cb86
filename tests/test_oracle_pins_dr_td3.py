"""Pins for the oracle parts round 1 left unpinned (-m "not gpu"):

* the domain-randomisation map or_effective_params (Q19, BASELINE configs[2]): each factor is
  checked through closed forms of the dynamics it must scale;
* the TD3 target (Q33; the clipped double-Q and the target-policy smoothing clip of the cited
  algorithm): targets built from constant / linear networks whose outputs are
  known in closed form;
* Adam's bias correction at t > 1 (Q34): with a constant gradient the bias-corrected moments
  are exactly g and g^2 at every t, so every step is -lr g / (|g| + eps);
* the fp16 rounding-midpoint margin of the MLP parity exclusion (SURVEY 8(c) parity test 5):
  brute force over numpy's float16 neighbours, and closed forms at binade edges.

Each check compares against something other than the oracle's own formula."""
import math

import numpy as np
import pytest

import inputs
import oracle

P = inputs.CRAZYFLIE
G = P["gravity"]
L = 0.028  # rotor arm (inputs.CRAZYFLIE rotor_pos)


def hover_rpm(c2=P["thrust_c"][2], m=P["mass"]):
    return math.sqrt(m * G / (4 * c2))


def state_with_thrusts(f, c2=P["thrust_c"][2]):
    """Level state at rest whose rotor speeds produce thrusts f (c0 = c1 = 0)."""
    s = np.zeros(17)
    s[3] = 1.0
    s[13:17] = np.sqrt(np.asarray(f) / c2)
    return s


def deriv(cfg, dr, s):
    p = oracle.effective_params(cfg, dr)
    return oracle.derivative(p, s, s[13:17], np.zeros(6))


# ---------------------------------------------------------------- DR effective parameters (Q19)
def test_dr_mass_factor_scales_linear_acceleration_only():
    """Mass factor 2 at the nominal hover speed: thrust m g against mass 2m gives v'_z = -g/2
    (Newton); no angular acceleration."""
    cfg = inputs.base_config()
    s = state_with_thrusts([P["mass"] * G / 4] * 4)
    ds = deriv(cfg, [2.0, 1, 1, 1, 1], s)
    assert abs(ds[9] - (-G / 2)) <= 1e-12
    assert np.all(np.abs(ds[10:13]) <= 1e-9)
    ds1 = deriv(cfg, [1.0, 1, 1, 1, 1], s)
    assert abs(ds1[9]) <= 1e-12


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("k", [0.8, 1.2, 2.0])
def test_dr_inertia_factor_scales_its_own_axis(axis, k):
    """Single-axis torque cases (roll / pitch / yaw closed forms): the J_ii factor
    divides only omega'_i; the other two factors leave it unchanged."""
    fh, d = P["mass"] * G / 4, 1e-4
    if axis == 0:   # roll: rotors 2, 3 (y = +l) up, 0, 1 (y = -l) down
        f, want = [fh - d, fh - d, fh + d, fh + d], 4 * L * d / P["J"][0]
    elif axis == 1:  # pitch: rotors 0, 3 (x = +l) up -> tau_y = -4 l d
        f, want = [fh + d, fh - d, fh - d, fh + d], -4 * L * d / P["J"][1]
    else:            # yaw: spin (-1, +1, -1, +1) -> tau_z = 4 c_tau d
        f, want = [fh - d, fh + d, fh - d, fh + d], 4 * P["torque_c"] * d / P["J"][2]
    cfg = inputs.base_config()
    s = state_with_thrusts(f)
    for j in range(3):
        dr = [1.0] * 5
        dr[1 + j] = k
        ds = deriv(cfg, dr, s)
        exp = want / k if j == axis else want
        assert abs(ds[10 + axis] - exp) <= 1e-9 * abs(want), (axis, j, ds[10 + axis], exp)
        others = [i for i in range(3) if i != axis]
        assert np.all(np.abs(ds[10 + np.array(others)]) <= 1e-9 * abs(want))


def test_dr_inertia_factors_in_the_gyroscopic_term():
    """Torque-free rotation (equal thrusts): Euler's equations J_x w_x' = (J_y - J_z) w_y w_z
    etc. with the randomised J = diag(k_x J_x, k_y J_y, k_z J_z) (textbook rigid body)."""
    cfg = inputs.base_config()
    s = state_with_thrusts([P["mass"] * G / 4] * 4)
    w = np.array([3.0, -5.0, 7.0])
    s[10:13] = w
    kx, ky, kz = 0.8, 1.15, 1.2
    ds = deriv(cfg, [1.0, kx, ky, kz, 1.0], s)
    Jx, Jy, Jz = kx * P["J"][0], ky * P["J"][1], kz * P["J"][2]
    exp = [(Jy - Jz) * w[1] * w[2] / Jx, (Jz - Jx) * w[2] * w[0] / Jy, (Jx - Jy) * w[0] * w[1] / Jz]
    assert np.allclose(ds[10:13], exp, rtol=1e-12, atol=0)


def test_dr_thrust_factor_scales_every_thrust_coefficient():
    """f = k (c0 + c1 w + c2 w^2) (P:57 thrust curve, Q19): with c0, c1, c2 all non-zero the
    vertical acceleration at a level state is 4 k f(w)/m - g and the yaw torque scales by k."""
    cfg = inputs.base_config()
    c = [0.01, 2e-6, 3.16e-10]
    cfg["params"]["thrust_c"] = c
    w = 12000.0
    f = c[0] + c[1] * w + c[2] * w * w
    s = np.zeros(17)
    s[3] = 1.0
    s[13:17] = w
    for k in (0.8, 1.0, 1.17):
        ds = deriv(cfg, [1, 1, 1, 1, k], s)
        assert abs(ds[9] - (4 * k * f / P["mass"] - G)) <= 1e-12 * G, k
    # yaw: two rotors of spin +1 faster; tau_z = c_tau (f(w+) - f(w-)) * 2 scales with k
    s[13:17] = [w, w + 500, w, w + 500]
    fp = c[0] + c[1] * (w + 500) + c[2] * (w + 500) ** 2
    for k in (0.8, 1.2):
        ds = deriv(cfg, [1, 1, 1, 1, k], s)
        exp = k * P["torque_c"] * 2 * (fp - f) / P["J"][2]
        assert abs(ds[12] - exp) <= 1e-9 * abs(exp), k


# ---------------------------------------------------------------- TD3 target (Q33)
IN = 18 + 4 * 4


def _offsets(in_dim=IN):
    na, nc = oracle.net_size(in_dim, 64, 4), oracle.net_size(32, 64, 1)
    o = {"actor": 0, "actor_t": na, "q1": 2 * na, "q2": 2 * na + nc, "q1_t": 2 * na + 2 * nc,
         "q2_t": 2 * na + 3 * nc, "na": na, "nc": nc}
    o["m_actor"] = 2 * na + 4 * nc
    o["v_actor"] = o["m_actor"] + na
    o["m_q1"] = o["v_actor"] + na
    o["v_q1"] = o["m_q1"] + nc
    o["m_q2"] = o["v_q1"] + nc
    o["v_q2"] = o["m_q2"] + nc
    return o


def _net_slices(n_in, n_out):
    """(W1, b1, W2, b2, W3, b3) offsets inside one net (layout [W1 b1 W2 b2 W3 b3])."""
    sizes = [64 * n_in, 64, 64 * 64, 64, n_out * 64, n_out]
    return np.concatenate([[0], np.cumsum(sizes)])


def _batch(B, seed=1, in_dim=IN):
    g = np.random.default_rng(seed)
    return {"o_a": g.normal(0, 0.5, (B, in_dim)), "o_c": g.normal(0, 0.5, (B, 28)),
            "a": g.uniform(-1, 1, (B, 4)), "r": g.normal(-1, 1, B), "o_a2": g.normal(0, 0.5, (B, in_dim)),
            "o_c2": g.normal(0, 0.5, (B, 28)), "done": (g.uniform(0, 1, B) < 0.3).astype(float),
            "eps": g.normal(0, 1, (B, 4))}


FROZEN = {"lr_actor": 0.0, "lr_critic": 0.0}


@pytest.mark.parametrize("K1,K2", [(3.0, 5.0), (5.0, 3.0), (-2.0, 4.0), (1.5, 1.5)])
def test_td3_target_uses_the_smaller_target_critic(K1, K2):
    """Clipped double-Q: with constant target critics Q1' = K1, Q2' = K2 (all weights 0,
    output bias K) and online critics that output 0, each critic loss is mean(y^2) with
    y = r + gamma (1 - done) min(K1, K2)."""
    o = _offsets()
    sl = _net_slices(32, 1)
    P = np.zeros(oracle.td3_block_size(IN))
    P[o["q1_t"] + sl[5]] = K1
    P[o["q2_t"] + sl[5]] = K2
    b = _batch(64)
    losses, _ = oracle.td3_update(P, IN, b, FROZEN, update_actor=False)
    y = b["r"] + 0.99 * (1 - b["done"]) * min(K1, K2)
    assert np.isclose(losses[0], np.mean(y ** 2), rtol=1e-13)
    assert np.isclose(losses[1], np.mean(y ** 2), rtol=1e-13)


def _linear_action_critic(P, base, w):
    """Critic q(o_c, a) = w . a: hidden units j < 4 carry a_j + 10 (> 0, so the ReLUs pass
    them), the output subtracts the offsets."""
    sl = _net_slices(32, 1)
    W1 = np.zeros((64, 32))
    b1 = np.zeros(64)
    W2 = np.zeros((64, 64))
    for j in range(4):
        W1[j, 28 + j] = 1.0
        b1[j] = 10.0
        W2[j, j] = 1.0
    W3 = np.zeros(64)
    W3[:4] = w
    P[base + sl[0]:base + sl[1]] = W1.ravel()
    P[base + sl[1]:base + sl[2]] = b1
    P[base + sl[2]:base + sl[3]] = W2.ravel()
    P[base + sl[4]:base + sl[5]] = W3
    P[base + sl[5]] = -10.0 * float(np.sum(w))


def test_td3_target_policy_smoothing_is_clipped():
    """a' = clip(pi'(o') + clip(sigma_t eps, -c_t, c_t), -1, 1): a constant target
    actor pi' = a0 (weights 0, b3 = atanh a0) and linear target critics q = e_k . a read each
    component of a' back through y = r + gamma a'_k (done = 0, online critics 0, B = 1)."""
    o = _offsets()
    sla = _net_slices(IN, 4)
    a0 = np.array([0.2, -0.5, 0.95, 0.0])
    eps = np.array([1.0, -1.0, 0.3, -2.0])
    sigma, clip = 10.0, 0.1
    want = np.clip(a0 + np.clip(sigma * eps, -clip, clip), -1, 1)  # (0.3, -0.6, 1.0, -0.1)
    b = _batch(1)
    b["eps"][0] = eps
    b["done"][0] = 0.0
    b["r"][0] = 50.0
    got = np.zeros(4)
    for k in range(4):
        P = np.zeros(oracle.td3_block_size(IN))
        P[o["actor_t"] + sla[5]:o["actor_t"] + sla[6]] = np.arctanh(a0)
        e = np.zeros(4)
        e[k] = 1.0
        _linear_action_critic(P, o["q1_t"], e)
        _linear_action_critic(P, o["q2_t"], e)
        losses, _ = oracle.td3_update(P, IN, b, {**FROZEN, "sigma_t": sigma, "clip_t": clip}, update_actor=False)
        got[k] = (math.sqrt(losses[0]) - 50.0) / 0.99
    assert np.allclose(got, want, atol=1e-12), (got, want)
    # unclipped: small sigma -> a' = a0 + sigma eps exactly
    b["eps"][0] = [0.1, -0.2, 0.0, 0.3]
    P = np.zeros(oracle.td3_block_size(IN))
    P[o["actor_t"] + sla[5]:o["actor_t"] + sla[6]] = np.arctanh(a0)
    _linear_action_critic(P, o["q1_t"], np.ones(4))
    _linear_action_critic(P, o["q2_t"], np.ones(4))
    losses, _ = oracle.td3_update(P, IN, b, {**FROZEN, "sigma_t": 0.2, "clip_t": 0.5}, update_actor=False)
    assert abs((math.sqrt(losses[0]) - 50.0) / 0.99 - np.sum(a0 + 0.2 * b["eps"][0])) <= 1e-12


# ---------------------------------------------------------------- Adam at t > 1 (Q34)
def _make_block(seed=0):
    g = np.random.default_rng(seed)
    P = np.zeros(oracle.td3_block_size(IN))
    o = _offsets()
    n_nets = o["m_actor"]
    P[:n_nets] = g.uniform(-0.2, 0.2, n_nets)
    return P


@pytest.mark.parametrize("t", [2, 3, 10])
def test_adam_bias_correction_at_step_t(t):
    """Moments prepared as t - 1 Adam steps of the same gradient g leave them at
    m = (1 - b1^(t-1)) g, v = (1 - b2^(t-1)) g^2 (geometric sums); step t then gives
    m_t = (1 - b1^t) g, v_t = (1 - b2^t) g^2 and, after bias correction, the step
    -lr g / (|g| + eps) (Kingma & Ba 2015)."""
    o = _offsets()
    b1, b2, lr, eps = 0.9, 0.999, 1e-3, 1e-8
    b = _batch(32, seed=4)
    P0 = _make_block()
    _, g = oracle.td3_update(P0.copy(), IN, b, FROZEN, update_actor=True, want_grads=True)
    nc, na = o["nc"], o["na"]
    g1, g2, ga = g[:nc], g[nc:2 * nc], g[2 * nc:]
    # critics (step t_critic = t); the actor is not updated
    P = P0.copy()
    for (m, v, gg) in (("m_q1", "v_q1", g1), ("m_q2", "v_q2", g2)):
        P[o[m]:o[m] + nc] = (1 - b1 ** (t - 1)) * gg
        P[o[v]:o[v] + nc] = (1 - b2 ** (t - 1)) * gg * gg
    oracle.td3_update(P, IN, b, {"lr_critic": lr, "lr_actor": 0.0}, t_critic=t, update_actor=False)
    for (q, m, v, gg) in (("q1", "m_q1", "v_q1", g1), ("q2", "m_q2", "v_q2", g2)):
        d = P[o[q]:o[q] + nc] - P0[o[q]:o[q] + nc]
        assert np.allclose(d, -lr * gg / (np.abs(gg) + eps), rtol=1e-9, atol=1e-15), (q, t)
        assert np.allclose(P[o[m]:o[m] + nc], (1 - b1 ** t) * gg, rtol=1e-12, atol=1e-300)
        assert np.allclose(P[o[v]:o[v] + nc], (1 - b2 ** t) * gg * gg, rtol=1e-12, atol=1e-300)
    # actor (step t_actor = t; critics frozen, so the actor gradient is the one measured above;
    # tau = 0 keeps the targets)
    P = P0.copy()
    P[o["m_actor"]:o["m_actor"] + na] = (1 - b1 ** (t - 1)) * ga
    P[o["v_actor"]:o["v_actor"] + na] = (1 - b2 ** (t - 1)) * ga * ga
    oracle.td3_update(P, IN, b, {"lr_critic": 0.0, "lr_actor": lr, "tau": 0.0}, t_actor=t, update_actor=True)
    d = P[:na] - P0[:na]
    assert np.allclose(d, -lr * ga / (np.abs(ga) + eps), rtol=1e-9, atol=1e-15), t


# ---------------------------------------------------------------- fp16 midpoint margin
def _brute_margin(v):
    """Relative distance of v to the nearest fp16 rounding midpoint, from numpy's float16
    neighbours of the rounded value (no exponent arithmetic)."""
    v = float(v)
    if v == 0.0:
        return math.inf
    h = np.float16(abs(v))
    lo = np.nextafter(h, np.float16(0))
    hi = np.nextafter(h, np.float16(np.inf))
    mids = [(float(h) + float(hi)) / 2]
    if float(h) > 0:
        mids.append((float(h) + float(lo)) / 2)
    return min(abs(abs(v) - m) for m in mids) / abs(v)


def _zero_policy(in_dim):
    z = lambda *s: np.zeros(s, dtype=np.uint16)  # noqa: E731  (fp16 +0 bit patterns)
    return {"W1": z(64, in_dim), "b1": z(64), "W2": z(64, 64), "b2": z(64), "W3": z(4, 64), "b3": z(4)}


@pytest.mark.parametrize("v,want", [
    (1.0 + 1e-4, (1e-4 + 2.0 ** -12) / (1.0 + 1e-4)),          # just above a binade edge
    (1.0 - 1e-5, (2.0 ** -12 - 1e-5) / (1.0 - 1e-5)),           # just below it
    (1.5 + 3e-4, (2.0 ** -11 - 3e-4) / (1.5 + 3e-4)),           # mid-binade, above the midpoint side
    (1000.4 * 2.0 ** -24, 0.1 / 1000.4),                       # subnormal: 1000.4 quanta of 2^-24, 0.1 from 1000.5
])
def test_midpoint_margin_closed_forms(v, want):
    """With a zero policy only the observation is quantised, so the margin is that of the
    smallest-margin observation; the other entries are exact halves with larger margins."""
    obs = np.full(18, 1.0 + 2.0 ** -10)  # margin 2^-11 / (1 + 2^-10) = 4.88e-4
    obs[5] = v
    m = oracle.mlp_midpoint_margin(oracle.PolicyHandle(_zero_policy(18)), obs)
    assert abs(m - want) <= 1e-12 * want, (m, want)
    assert abs(_brute_margin(v) - want) <= 1e-12 * want


def test_midpoint_margin_matches_brute_force_on_realistic_inputs():
    """Every quantisation point of the MLP (observation, positive layer-1 and layer-2
    pre-activations from numpy's matmul on the fp16-decoded operands) against the float16
    neighbour brute force; the oracle's margin is their minimum."""
    W = inputs.policy_weights(146, 64, seed=7)
    ph = oracle.PolicyHandle(W)
    dec = {k: v.view(np.float16).astype(np.float64) for k, v in W.items()}
    g = np.random.default_rng(3)
    for trial in range(60):
        obs = np.concatenate([g.normal(0, 0.5, 18), g.uniform(-1, 1, 128)])
        x0 = obs.astype(np.float16).astype(np.float64)
        a1 = dec["W1"] @ x0 + dec["b1"]
        h1 = np.maximum(a1, 0).astype(np.float16).astype(np.float64)
        a2 = dec["W2"] @ h1 + dec["b2"]
        pts = list(obs) + [x for x in a1 if x > 0] + [x for x in a2 if x > 0]
        want = min(_brute_margin(x) for x in pts)
        got = oracle.mlp_midpoint_margin(ph, obs)
        assert abs(got - want) <= 1e-9 * want + 1e-14, (trial, got, want)
