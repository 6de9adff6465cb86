"""Pins for the FP64 oracle (-m "not gpu").

Every check here compares the oracle against something other than itself: values the paper
prints, closed forms, textbook identities, library routines (numpy float16, numpy matmul),
brute force on tiny inputs, or statistics.  Each test names the passage it pins.
"""
import json
import math
import os

import numpy as np
import pytest

import inputs
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
P = inputs.CRAZYFLIE


def _params(**over):
    d = dict(P)
    d.update(over)
    return oracle.params_struct(d)


def hover_rpm(p=P):
    # Closed form of thrust balance 4 c2 w^2 = m g for c0 = c1 = 0
    return math.sqrt(p["mass"] * p["gravity"] / (4 * p["thrust_c"][2]))


def hover_state(p=P):
    s = np.zeros(17)
    s[3] = 1.0
    s[13:17] = hover_rpm(p)
    return s


# ---------------------------------------------------------------- Philox (Q20)
def test_philox_kat_random123():
    rows = [l.split() for l in open(os.path.join(GOLD, "philox_kat.txt")) if l.strip() and l[0] != "#"]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        out = oracle.philox(v[0:4], v[4:6])
        assert list(out) == v[6:10]


def test_uniform_range_and_resolution():
    assert oracle.uniform(0) == 0.5 / 2 ** 23
    assert oracle.uniform(0xFFFFFFFF) == 1 - 0.5 / 2 ** 23
    # every uniform is exactly representable in fp32 (Q20)
    for x in (0, 511, 512, 0x80000000, 0xFFFFFE00, 0xFFFFFFFF, 123456789):
        u = oracle.uniform(x)
        assert float(np.float32(u)) == u
    assert 0 < oracle.uniform(12345678) < 1


def test_box_muller_moments():
    g = np.random.default_rng(0)
    xs = g.integers(0, 2 ** 32, (20000, 2), dtype=np.uint64)
    z = np.array([oracle.box_muller(a, b) for a, b in xs]).ravel()
    n = z.size
    assert abs(z.mean()) < 4 / math.sqrt(n)
    assert abs(z.var() - 1) < 4 * math.sqrt(2 / n)
    # 4th moment of N(0,1) is 3
    assert abs((z ** 4).mean() - 3) < 0.15


# ---------------------------------------------------------------- fp16 rounding (Q21)
def test_q16_matches_numpy_float16():
    g = np.random.default_rng(1)
    x = np.concatenate([
        g.standard_normal(3000) * 10.0 ** g.integers(-9, 5, 3000),
        [0.0, -0.0, 1.0, 65504.0, 65519.99, 65520.0, -70000.0, 6.1e-5, 5.96e-8, 2.98e-8, 2.99e-8, 1e-9],
    ])
    # exact rounding midpoints between neighbouring halves (ties-to-even)
    h = np.arange(0, 0x7BFF, 97, dtype=np.uint16).view(np.float16).astype(np.float64)
    h2 = np.arange(1, 0x7C00, 97, dtype=np.uint16).view(np.float16).astype(np.float64)
    mids = (h[: len(h2)] + h2[: len(h)]) / 2
    x = np.concatenate([x, mids, -mids])
    with np.errstate(over="ignore"):
        ref = x.astype(np.float16).astype(np.float64)
    got = oracle.q16(x)
    assert np.array_equal(got, ref)


def test_half_to_double_matches_numpy():
    bits = np.arange(0, 65536, 7, dtype=np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = oracle.half_to_double(bits)
    fin = np.isfinite(ref)
    assert np.array_equal(got[fin], ref[fin])
    assert np.array_equal(np.isnan(got), np.isnan(ref))


# ---------------------------------------------------------------- rotation
def test_rotation_special_cases():
    assert np.array_equal(oracle.rotation([1, 0, 0, 0]), np.eye(3))
    assert np.allclose(oracle.rotation([0, 0, 0, 1]), np.diag([-1, -1, 1]), atol=0)


def test_rotation_orthonormal_det_double_cover_rodrigues():
    g = np.random.default_rng(2)
    for _ in range(200):
        q = g.standard_normal(4)
        q /= np.linalg.norm(q)
        R = oracle.rotation(q)
        assert np.allclose(R.T @ R, np.eye(3), atol=1e-12)
        assert abs(np.linalg.det(R) - 1) < 1e-12
        assert np.array_equal(R, oracle.rotation(-q))  # double cover, bitwise
        # Rodrigues: R = I + sin(th) K + (1 - cos(th)) K^2 for axis n, angle th
        th = 2 * math.atan2(np.linalg.norm(q[1:]), q[0])
        n = q[1:] / np.linalg.norm(q[1:])
        K = np.array([[0, -n[2], n[1]], [n[2], 0, -n[0]], [-n[1], n[0], 0]])
        Rr = np.eye(3) + math.sin(th) * K + (1 - math.cos(th)) * K @ K
        assert np.allclose(R, Rr, atol=1e-12)


# ---------------------------------------------------------------- dynamics
def test_hover_derivative_is_zero():
    s = hover_state()
    ds = oracle.derivative(_params(), s, s[13:17], np.zeros(6))
    assert np.max(np.abs(ds)) <= 1e-12


def test_free_fall_derivative():
    s = np.zeros(17)
    s[3] = 1.0
    ds = oracle.derivative(_params(), s, np.zeros(4), np.zeros(6))
    assert np.array_equal(ds[7:10], [0, 0, -P["gravity"]])
    assert np.array_equal(ds[10:13], [0, 0, 0])


def test_thrust_direction_tilted():
    # rotation about x by th: R e_z = (0, -sin th, cos th); v' = R e_z T/m - g e_z
    th = 0.3
    s = hover_state()
    s[3:7] = [math.cos(th / 2), math.sin(th / 2), 0, 0]
    ds = oracle.derivative(_params(), s, s[13:17], np.zeros(6))
    T = 4 * P["thrust_c"][2] * hover_rpm() ** 2
    exp = np.array([0, -math.sin(th), math.cos(th)]) * T / P["mass"] - np.array([0, 0, P["gravity"]])
    assert np.allclose(ds[7:10], exp, rtol=1e-12, atol=1e-12)


def _rpm_for(f):
    return np.sqrt(np.asarray(f) / P["thrust_c"][2])


def test_roll_torque_closed_form():
    l = 0.028
    fh = P["mass"] * P["gravity"] / 4
    d = 0.1 * fh
    s = hover_state()
    s[13:17] = _rpm_for([fh - d, fh - d, fh + d, fh + d])
    ds = oracle.derivative(_params(), s, s[13:17], np.zeros(6))
    assert abs(ds[10] - 4 * l * d / P["J"][0]) < 1e-9 * abs(ds[10])
    assert abs(ds[11]) < 1e-9 and abs(ds[12]) < 1e-9
    # roll rate grows linearly: RK4 exact for linear-in-time omega_x with constant torque
    # (omega = (wx,0,0) has no gyroscopic term); after n steps omega_x = n dt * alpha
    pr = _params()
    x = s.copy()
    for _ in range(10):
        x = oracle.rk4(pr, x, x[13:17], np.zeros(6), 0.01)
    assert abs(x[10] - 0.1 * ds[10]) < 1e-12 * abs(ds[10]) + 1e-12
    # attitude after 0.1 s: angle = alpha t^2 / 2 about x
    ang = 0.5 * ds[10] * 0.1 ** 2
    assert np.allclose(x[3:7] / np.linalg.norm(x[3:7]), [math.cos(ang / 2), math.sin(ang / 2), 0, 0], atol=1e-10)


def test_yaw_torque_closed_form():
    fh = P["mass"] * P["gravity"] / 4
    d = 0.1 * fh
    s = hover_state()
    s[13:17] = _rpm_for([fh - d, fh + d, fh - d, fh + d])
    ds = oracle.derivative(_params(), s, s[13:17], np.zeros(6))
    assert abs(ds[12] - 4 * P["torque_c"] * d / P["J"][2]) < 1e-9 * abs(ds[12])
    assert abs(ds[10]) < 1e-9 and abs(ds[11]) < 1e-9


def test_gyroscopic_term_sign():
    # Euler's equations: J w' = -w x (J w).  With w = (a, b, 0):
    # w x Jw = (0, 0, a b (Jy - Jx)) -> wz' = -a b (Jy - Jx) / Jz
    J = [2e-6, 5e-6, 7e-6]
    pr = _params(J=J, thrust_c=[0, 0, 0])
    s = np.zeros(17)
    s[3] = 1
    a, b = 3.0, -2.0
    s[10:13] = [a, b, 0]
    ds = oracle.derivative(pr, s, np.zeros(4), np.zeros(6))
    assert abs(ds[12] - (-a * b * (J[1] - J[0]) / J[2])) < 1e-9
    assert abs(ds[10]) < 1e-12 and abs(ds[11]) < 1e-12


def test_quaternion_kinematics_body_rate():
    # constant body rate with isotropic J and no thrust: q(t) = q0 (x) exp(w t / 2)
    pr = _params(J=[4e-6, 4e-6, 4e-6], thrust_c=[0, 0, 0], rpm_min=0.0)
    g = np.random.default_rng(3)
    q0 = g.standard_normal(4)
    q0 /= np.linalg.norm(q0)
    w = np.array([1.3, -0.7, 2.1])
    s = np.zeros(17)
    s[3:7] = q0
    s[10:13] = w
    x = s.copy()
    for _ in range(100):
        x = oracle.rk4(pr, x, np.zeros(4), np.zeros(6), 0.01)
    t = 1.0
    nw = np.linalg.norm(w)
    e = np.concatenate([[math.cos(nw * t / 2)], math.sin(nw * t / 2) * w / nw])
    qw, qx, qy, qz = q0
    ew, ex, ey, ez = e
    ref = np.array([qw * ew - qx * ex - qy * ey - qz * ez,
                    qw * ex + qx * ew + qy * ez - qz * ey,
                    qw * ey - qx * ez + qy * ew + qz * ex,
                    qw * ez + qx * ey - qy * ex + qz * ew])
    assert np.allclose(x[3:7], ref, atol=1e-8)


def test_disturbance_enters_linearly():
    s = hover_state()
    dist = np.array([0.01, -0.02, 0.005, 1e-5, -2e-5, 3e-5])
    d0 = oracle.derivative(_params(), s, s[13:17], np.zeros(6))
    d1 = oracle.derivative(_params(), s, s[13:17], dist)
    assert np.allclose(d1[7:10] - d0[7:10], dist[:3] / P["mass"], rtol=1e-12, atol=1e-15)
    assert np.allclose(d1[10:13] - d0[10:13], dist[3:] / np.array(P["J"]), rtol=1e-12)


# ---------------------------------------------------------------- motor lag
def test_motor_lag_discrete_closed_form_and_63_percent():
    gold = json.load(open(os.path.join(GOLD, "paper_constants.json")))
    Tm = gold["motor_time_constant_s"]["value"]
    dt = 1.0 / gold["sim_rate_hz"]["value"]
    pr = _params(motor_tau=Tm)
    u = 12000.0
    s = np.zeros(17)
    s[3] = 1
    h = dt / Tm
    rho = 1 - h + h ** 2 / 2 - h ** 3 / 6 + h ** 4 / 24
    x = s.copy()
    n = int(round(Tm / dt))
    for k in range(1, n + 1):
        x = oracle.rk4(pr, x, np.full(4, u), np.zeros(6), dt)
        x[3:7] = [1, 0, 0, 0]
        x[0:3] = 0
        x[7:13] = 0
        assert np.allclose(x[13:17], u * (1 - rho ** k), rtol=1e-13)
    frac = x[13] / u
    ref = gold["rc_step_response_fraction"]
    assert abs(frac - ref["value"]) <= ref["tolerance_rel"] * ref["value"]


# ---------------------------------------------------------------- RK4 (Q1)
def test_free_fall_one_second():
    cfg = inputs.config_c1()
    env = oracle.new_envs(1)
    env[0]["s"][3] = 1.0
    env[0]["dr"][:] = 1.0
    for t in range(100):
        oracle.env_step(cfg, env, 0, t, [-1, -1, -1, -1])  # a = -1 -> rpm_min = 0
    assert abs(env[0]["s"][2] - (-0.5 * P["gravity"])) < 1e-6
    assert abs(env[0]["s"][9] - (-P["gravity"])) < 1e-9


def test_rk4_fourth_order_convergence():
    pr = _params()
    g = np.random.default_rng(4)
    s0 = hover_state()
    s0[10:13] = [0.5, -0.3, 0.2]
    s0[7:10] = [0.2, 0.1, -0.1]
    u = hover_rpm() * np.array([1.01, 0.99, 1.02, 0.98])

    def run(dt, T=0.32):
        x = s0.copy()
        for _ in range(int(round(T / dt))):
            x = oracle.rk4(pr, x, u, np.zeros(6), dt)
        return x

    ref = run(0.0025 / 16)
    e = [np.max(np.abs(run(dt) - ref)[:13]) for dt in (0.02, 0.01, 0.005)]
    r1, r2 = e[0] / e[1], e[1] / e[2]
    assert 12 < r1 < 20 and 12 < r2 < 20, (e, r1, r2)


def test_hover_state_unchanged_by_step():
    pr = _params()
    s = hover_state()
    x = oracle.project(pr, oracle.rk4(pr, s, s[13:17], np.zeros(6), 0.01))
    assert np.max(np.abs(x - s)) <= 1e-9 * max(1, hover_rpm())


# ---------------------------------------------------------------- action map
def test_action_map():
    pr = _params(rpm_min=1000.0)
    assert oracle.action_to_rpm(pr, -1) == 1000.0
    assert oracle.action_to_rpm(pr, 1) == P["rpm_max"]
    assert abs(oracle.action_to_rpm(pr, 0) - (1000.0 + P["rpm_max"]) / 2) < 1e-9


# ---------------------------------------------------------------- reward
def test_reward_special_cases():
    cfg = inputs.base_config()
    w, _ = oracle.stage(cfg, 0)
    cr = cfg["curriculum"]["init"]
    s = np.zeros(17)
    s[3] = 1
    assert oracle.reward(w, s, cr["C_rab"]) == cr["C_rs"]
    s2 = s.copy()
    s2[3:7] = [0, 1, 0, 0]  # q_w = 0: 180 deg
    assert abs(oracle.reward(w, s2, cr["C_rab"]) - (cr["C_rs"] - cr["C_rq"])) < 1e-15
    g = np.random.default_rng(5)
    for _ in range(100):
        x = g.standard_normal(17)
        x[3:7] /= np.linalg.norm(x[3:7])
        a = g.uniform(-1, 1, 4)
        r = oracle.reward(w, x, a)
        assert r <= cr["C_rs"]
        y = x.copy()
        y[3:7] *= -1
        assert oracle.reward(w, y, a) == r  # depends on q_w^2 only
        # term-by-term: scaling p by 2 quadruples the position penalty
        z = x.copy()
        z[0:3] *= 2
        assert abs((oracle.reward(w, z, a) - r) - (-3 * cr["C_rp"] * np.sum(x[0:3] ** 2))) < 1e-12


# ---------------------------------------------------------------- curriculum
def test_curriculum_closed_form_and_saturation():
    cfg = inputs.base_config()
    cur = cfg["curriculum"]
    I = cur["interval"]
    for k in range(0, 12):
        w, sg = oracle.stage(cfg, k * I + (I // 2))
        exp_p = min(cur["init"]["C_rp"] * cur["factor"]["C_rp"] ** k, cur["target"]["C_rp"])
        exp_a = min(cur["init"]["C_ra"] * cur["factor"]["C_ra"] ** k, cur["target"]["C_ra"])
        exp_s = max(cur["sigma_init"] * cur["sigma_factor"] ** k, cur["sigma_target"])
        assert abs(w.C_rp - exp_p) <= 1e-12 * exp_p
        assert abs(w.C_ra - exp_a) <= 1e-12 * exp_a
        assert abs(sg - exp_s) <= 1e-12 * exp_s
        assert w.C_rq == cur["init"]["C_rq"]  # factor 1 -> constant
    w, sg = oracle.stage(cfg, 1000 * I)
    assert w.C_rp == cur["target"]["C_rp"] and w.C_ra == cur["target"]["C_ra"]
    assert sg == cur["sigma_target"]
    # stage boundary: t = I - 1 is stage 0, t = I is stage 1
    assert oracle.stage(cfg, I - 1)[0].C_rp == cur["init"]["C_rp"]
    assert oracle.stage(cfg, I)[0].C_rp == cur["init"]["C_rp"] * cur["factor"]["C_rp"]


# ---------------------------------------------------------------- termination
def _step_from(cfg, s, a):
    env = oracle.new_envs(1)
    env[0]["s"] = s
    env[0]["dr"][:] = 1
    so = oracle.env_step(cfg, env, 0, 0, a)
    return so, env


def test_termination_box():
    cfg = inputs.base_config(flags=inputs.TERMINATION)
    ah = np.full(4, 2 * hover_rpm() / P["rpm_max"] - 1)
    s = hover_state()
    so, _ = _step_from(cfg, s, ah)
    assert so.flags == 0
    s1 = s.copy()
    s1[0] = 0.6  # exactly on the bound: strict inequality -> not terminated
    so, env = _step_from(cfg, s1, ah)
    assert env[0]["s"][0] == 0.6 and so.flags == 0
    s2 = s.copy()
    s2[0] = 0.6 + 1e-9
    so, _ = _step_from(cfg, s2, ah)
    assert so.flags & oracle.FLAG_TERMINATED
    assert so.margin[0] > 0
    s3 = s.copy()
    s3[10] = 40.0
    so, _ = _step_from(cfg, s3, ah)
    assert so.flags & oracle.FLAG_TERMINATED and so.margin[2] > 0


def test_truncation_at_episode_cap():
    cfg = inputs.base_config(flags=inputs.TERMINATION, max_episode_steps=500)
    ah = np.full(4, 2 * hover_rpm() / P["rpm_max"] - 1)
    env = oracle.new_envs(1)
    env[0]["s"] = hover_state()
    env[0]["dr"][:] = 1
    for t in range(500):
        so = oracle.env_step(cfg, env, 0, t, ah)
        if t < 499:
            assert so.flags == 0
    assert so.flags == oracle.FLAG_TRUNCATED


def test_divergence_terminates():
    cfg = inputs.base_config(flags=0)
    s = hover_state()
    s[7] = np.nan
    so, _ = _step_from(cfg, s, np.zeros(4))
    assert so.flags & oracle.FLAG_DIVERGED and so.flags & oracle.FLAG_TERMINATED
    assert so.reward == 0.0


def test_hover_env_step_reward_is_survival():
    # hover action from hover state -> not done, r = C_rs when C_rab = hover action
    ah = 2 * hover_rpm() / P["rpm_max"] - 1
    cfg = inputs.base_config(flags=inputs.TERMINATION)
    cfg["curriculum"]["init"]["C_rab"] = [ah] * 4
    so, env = _step_from(cfg, hover_state(), np.full(4, ah))
    assert so.flags == 0
    assert abs(so.reward - cfg["curriculum"]["init"]["C_rs"]) < 1e-12
    assert np.max(np.abs(env[0]["s"] - hover_state())) < 1e-9 * hover_rpm()


# ---------------------------------------------------------------- reset
def test_reset_distribution_bounds_and_moments():
    cfg = inputs.base_config(flags=inputs.ALL_NO_DR | inputs.DOMAIN_RAND)
    n = 6000
    E = oracle.reset_many(cfg, np.arange(n), 7)
    s = E["s"]
    P0, V0, W0 = cfg["init_pos"], cfg["init_vel"], cfg["init_angvel"]
    assert np.all(np.abs(s[:, 0:3]) <= P0)
    assert np.all(np.abs(s[:, 7:10]) <= V0) and np.all(np.abs(s[:, 10:13]) <= W0)
    lo, hi = cfg["init_rpm"]
    assert np.all((s[:, 13:17] >= lo) & (s[:, 13:17] <= hi))
    assert np.allclose(np.linalg.norm(s[:, 3:7], axis=1), 1, atol=1e-12)
    ang = 2 * np.arccos(np.clip(s[:, 3], -1, 1))
    assert np.all(ang <= cfg["init_angle"] + 1e-12)
    # U[a,b]: mean (a+b)/2, var (b-a)^2/12
    for col, (a, b) in [(0, (-P0, P0)), (8, (-V0, V0)), (14, (lo, hi))]:
        x = s[:, col]
        se = (b - a) / math.sqrt(12 * n)
        assert abs(x.mean() - (a + b) / 2) < 4 * se
        assert abs(x.var() - (b - a) ** 2 / 12) < 0.06 * (b - a) ** 2 / 12
    # angle ~ U[0, theta_max]
    assert abs(ang.mean() - cfg["init_angle"] / 2) < 4 * cfg["init_angle"] / math.sqrt(12 * n)
    # uniform axis: mean of the axis vector ~ 0, E[z^2] = 1/3
    ax = s[:, 4:7] / np.linalg.norm(s[:, 4:7], axis=1, keepdims=True)
    assert np.all(np.abs(ax.mean(axis=0)) < 4 / math.sqrt(3 * n))
    assert abs((ax[:, 2] ** 2).mean() - 1 / 3) < 0.03
    # disturbance and DR bounds
    F, Tq = cfg["dist_force"], cfg["dist_torque"]
    d = E["dist"]
    assert np.all(np.abs(d[:, :3]) <= F) and np.all(np.abs(d[:, 3:]) <= Tq)
    assert abs(d[:, 0].var() - (2 * F) ** 2 / 12) < 0.06 * (2 * F) ** 2 / 12
    dr = E["dr"]
    assert np.all((dr >= 0.8) & (dr <= 1.2))
    assert abs(dr[:, 4].mean() - 1.0) < 4 * 0.4 / math.sqrt(12 * n)
    # history filled with the normalised initial rotor speeds (Q10)
    H = E["hist"]
    exp = 2 * (s[:, 13:17] - P["rpm_min"]) / (P["rpm_max"] - P["rpm_min"]) - 1
    assert np.allclose(H[:, 31, :], exp, atol=1e-15) and np.allclose(H[:, 0, :], exp, atol=1e-15)
    assert np.all(E["ep_step"] == 0) and np.all(E["ep_return"] == 0)


def test_reset_determinism_and_independence():
    cfg = inputs.base_config()
    a = oracle.reset(cfg, 5, 3)
    b = oracle.reset(cfg, 5, 3)
    c = oracle.reset(cfg, 6, 3)
    d = oracle.reset(cfg, 5, 4)
    assert a.tobytes() == b.tobytes()
    assert not np.array_equal(a["s"], c["s"]) and not np.array_equal(a["s"], d["s"])


def test_reset_zero_bounds_gives_identity_state():
    cfg = inputs.base_config(flags=0, init_pos=0.0, init_angle=0.0, init_vel=0.0, init_angvel=0.0,
                             init_rpm=[10000.0, 10000.0])
    e = oracle.reset(cfg, 0, 0)
    exp = np.zeros(17)
    exp[3] = 1
    exp[13:17] = 10000.0
    assert np.array_equal(e["s"], exp)
    assert np.array_equal(e["dist"], np.zeros(6)) and np.array_equal(e["dr"], np.ones(5))


# ---------------------------------------------------------------- observation
def test_observation_noise_free_and_dims():
    gold = json.load(open(os.path.join(GOLD, "paper_constants.json")))
    cfg = inputs.base_config(flags=0, n_hist=32)
    e = oracle.reset(cfg, 3, 0)
    o = oracle.observe(cfg, e, 3, 0)
    assert o.size == gold["actor_obs_dim_base"]["value"] + 4 * 32
    exp = np.concatenate([e["s"][0:3], oracle.rotation(e["s"][3:7]).ravel(), e["s"][7:10],
                          e["s"][10:13], e["hist"].ravel()])
    assert np.array_equal(o, exp)
    cfg0 = inputs.base_config(flags=0, n_hist=0)
    assert oracle.observe(cfg0, e, 3, 0).size == 18


def test_observation_noise_moments():
    cfg = inputs.base_config(flags=inputs.OBS_NOISE, obs_sigma=[0.1, 0.2, 0.3, 0.4])
    e = oracle.reset(inputs.base_config(flags=0), 0, 0)
    clean = oracle.observe(inputs.base_config(flags=0), e, 0, 0)[:18]
    n = 3000
    X = np.array([oracle.observe(cfg, e, 0, t)[:18] for t in range(n)]) - clean
    sig = np.array([0.1] * 3 + [0.2] * 9 + [0.3] * 3 + [0.4] * 3)
    assert np.all(np.abs(X.mean(axis=0)) < 4.5 * sig / math.sqrt(n))
    assert np.all(np.abs(X.std(axis=0) / sig - 1) < 0.1)
    # components are uncorrelated
    Cm = np.corrcoef((X / sig).T)
    assert np.max(np.abs(Cm - np.eye(18))) < 0.1


# ---------------------------------------------------------------- env step composition
def test_env_step_history_push_and_invariants():
    cfg = inputs.config_c2()
    e = oracle.reset_many(cfg, [9], 0)
    h0 = e[0]["hist"].copy()
    a = np.array([0.3, -0.2, 0.9, 2.0])
    so = oracle.env_step(cfg, e, 9, 0, a)
    if not (so.flags & oracle.FLAG_RESET):
        assert np.array_equal(e[0]["hist"][0], np.array(so.a_applied))
        assert np.array_equal(e[0]["hist"][1:], h0[:-1])
        assert abs(np.linalg.norm(e[0]["s"][3:7]) - 1) < 1e-14
    assert all(-1 <= x <= 1 for x in so.a_applied)


def test_action_noise_is_seeded_gaussian():
    cfg = inputs.base_config(flags=inputs.ACTION_NOISE)
    w, sg = oracle.stage(cfg, 0)
    n = 2000
    z = []
    for t in range(n):
        e = oracle.new_envs(1)
        e[0]["s"][3] = 1
        e[0]["dr"][:] = 1
        so = oracle.env_step(cfg, e, 1, t, np.zeros(4))
        z.append(np.array(so.a_applied) / sg)
    z = np.array(z).ravel()
    assert abs(z.mean()) < 4 / math.sqrt(z.size)
    assert abs(z.std() - 1) < 0.05


# ---------------------------------------------------------------- MLP (Q21)
def test_mlp_matches_numpy_on_quantised_operands():
    W = inputs.policy_weights(146, 64, seed=7)
    pol = oracle.PolicyHandle(W)
    f = lambda k: W[k].view(np.float16).astype(np.float64)  # noqa: E731
    g = np.random.default_rng(6)
    for _ in range(20):
        o = g.standard_normal(146) * 2
        x0 = o.astype(np.float16).astype(np.float64)
        h1 = np.maximum(f("W1") @ x0 + f("b1"), 0).astype(np.float16).astype(np.float64)
        h2 = np.maximum(f("W2") @ h1 + f("b2"), 0).astype(np.float16).astype(np.float64)
        a = np.tanh(f("W3") @ h2 + f("b3"))
        assert np.allclose(oracle.mlp(pol, o), a, rtol=1e-12, atol=1e-14)


def test_mlp_zero_weights_gives_tanh_bias():
    W = inputs.policy_weights(146, 64, seed=1, out_bias=0.5)
    for k in ("W1", "b1", "W2", "b2", "W3"):
        W[k] = np.zeros_like(W[k])
    pol = oracle.PolicyHandle(W)
    a = oracle.mlp(pol, np.ones(146))
    assert np.allclose(a, np.tanh(np.float64(np.float16(0.5))), rtol=1e-15)


# ---------------------------------------------------------------- rollout driver
def test_rollout_matches_stepwise_and_is_thread_invariant():
    cfg = inputs.config_c2()
    n, T = 24, 60
    ids = np.arange(100, 100 + n, dtype=np.uint64)
    E0 = oracle.reset_many(cfg, ids, 0)
    acts = inputs.actions_near_hover(T, n).transpose(0, 2, 1).copy()  # (T, n, 4)
    E1 = E0.copy()
    st1, tr1 = oracle.rollout(cfg, E1, ids, 0, T, oracle.MODE_ACTIONS, actions=acts, trace=True, nthreads=1)
    E2 = E0.copy()
    st2, _ = oracle.rollout(cfg, E2, ids, 0, T, oracle.MODE_ACTIONS, actions=acts, nthreads=4)
    assert E1.tobytes() == E2.tobytes()
    # per-thread partial sums are reduced in a fixed order; only the FP summation order differs
    assert np.array_equal(st1[[0, 1, 2, 3, 4, 7]], st2[[0, 1, 2, 3, 4, 7]])
    assert np.allclose(st1, st2, rtol=1e-12)
    E3 = E0.copy()
    st3 = np.zeros(8)
    for t in range(T):
        for i in range(n):
            e = E3[i:i + 1]
            oracle.env_step(cfg, e, int(ids[i]), t, acts[t, i], st3)
    assert E3.tobytes() == E1.tobytes() and np.allclose(st3, st1, rtol=1e-12)
    assert st1[7] == n * T
    # stats = sums over the episodes seen in the trace
    fl = tr1[:, :, 26].astype(int)
    ended = (fl & (oracle.FLAG_TERMINATED | oracle.FLAG_TRUNCATED)) != 0
    assert st1[0] == ended.sum()


# ---------------------------------------------------------------- NEXT f1/f2
def test_no_rotor_delay_sets_rotor_speed_to_setpoint():
    # with the rotor-delay switch off, omega_m equals the setpoint immediately
    cfg = inputs.base_config(flags=inputs.NO_ROTOR_DELAY)
    env = oracle.new_envs(1)
    env[0]["s"] = hover_state()
    env[0]["s"][13:17] = 1000.0
    env[0]["dr"][:] = 1
    a = np.array([0.3, -0.5, 0.9, -1.0])
    oracle.env_step(cfg, env, 0, 0, a)
    u = [oracle.action_to_rpm(_params(), x) for x in a]
    assert np.allclose(env[0]["s"][13:17], u, rtol=0, atol=1e-9)
    # and with the lag the rotors move only part of the way (63 % after T_m = 15 steps)
    cfg2 = inputs.base_config(flags=0)
    env2 = oracle.new_envs(1)
    env2[0]["s"] = hover_state()
    env2[0]["s"][13:17] = 1000.0
    env2[0]["dr"][:] = 1
    oracle.env_step(cfg2, env2, 0, 0, a)
    assert np.all(np.abs(env2[0]["s"][13:17] - 1000.0) < np.abs(np.array(u) - 1000.0) * 0.1)


def test_critic_observation():
    gold = json.load(open(os.path.join(GOLD, "paper_constants.json")))
    e = oracle.new_envs(1)[0]
    e["s"] = hover_state()
    o = oracle.critic_observe(e)
    assert o.size == gold["critic_obs_dim"]["value"]
    # hover at origin, zero disturbance -> (0^3, I, 0^3, 0^3, w_h 1^4, 0^3, 0^3)
    exp = np.concatenate([np.zeros(3), np.eye(3).ravel(), np.zeros(6), np.full(4, hover_rpm()), np.zeros(6)])
    assert np.allclose(o, exp, rtol=1e-15, atol=0)
    e2 = oracle.reset(inputs.config_c2(), 4, 2)
    o2 = oracle.critic_observe(e2)
    assert np.array_equal(o2[18:22], e2["s"][13:17]) and np.array_equal(o2[22:28], e2["dist"])
    assert np.allclose(o2[3:12].reshape(3, 3), oracle.rotation(e2["s"][3:7]))


def test_recompute_reward_matches_step_reward_and_stages():
    cfg = inputs.config_c2()
    cfg["curriculum"]["interval"] = 10
    e = oracle.reset_many(cfg, [3], 0)
    a = np.array([0.1, 0.2, 0.3, 0.4])
    so = oracle.env_step(cfg, e, 3, 25, a)
    assert oracle.recompute_reward(cfg, 25, so.final_s, so.a_applied) == so.reward
    # a later stage re-weights the same transition (P:231 recalculation after a curriculum change)
    w2, _ = oracle.stage(cfg, 95)
    assert oracle.recompute_reward(cfg, 95, so.final_s, so.a_applied) == oracle.reward(w2, so.final_s, so.a_applied)
    bad = np.array(so.final_s)
    bad[4] = np.nan
    assert oracle.recompute_reward(cfg, 25, bad, so.a_applied) == 0.0


# ---- f3: Lissajous tracking evaluation (Table III; Q28-Q31) -------------

def test_lissajous_reference_closed_forms():
    """p(t) = [cos(2 pi t/T), sin(4 pi t/T)/2, z]: the paper's special points, and the
    velocity pinned as the numerical derivative of the position (not a retyped formula)."""
    T, z = 5.5, 1.25
    p, v = oracle.lissajous(0.0, T, 1.0, 0.5, z)
    assert np.allclose(p, [1, 0, z], atol=1e-15) and np.allclose(v, [0, 2 * math.pi / T, 0], atol=1e-15)
    p, _ = oracle.lissajous(T / 2, T, 1.0, 0.5, z)
    assert np.allclose(p, [-1, 0, z], atol=1e-14)
    p, _ = oracle.lissajous(T / 4, T, 1.0, 0.5, z)
    assert np.allclose(p, [0, 0, z], atol=1e-14)  # the figure-eight crossing
    p, _ = oracle.lissajous(T / 8, T, 1.0, 0.5, z)
    assert np.isclose(p[1], 0.5, atol=1e-14)      # maximal y excursion = the amplitude 1/2
    rng = np.random.default_rng(3)
    for t in rng.uniform(0, 3 * T, 5):
        h = 1e-6
        pp, v = oracle.lissajous(t, T)
        fd = (oracle.lissajous(t + h, T)[0] - oracle.lissajous(t - h, T)[0]) / (2 * h)
        assert np.allclose(v, fd, atol=1e-8)
    # peak speed of the fast (3.5 s) trajectory: order of the paper's "up to 3 m/s"
    sp = max(np.linalg.norm(oracle.lissajous(t, 3.5)[1]) for t in np.linspace(0, 3.5, 701))
    assert 2.0 < sp < 3.5


def test_setpoint_shift_identity_and_clipping():
    cfg = inputs.config_c4()
    e = oracle.reset(cfg, 7, 0)
    o = oracle.observe(cfg, e, 7, 5)
    # zero reference: identity (as long as the observation is inside the bounds)
    z3 = np.zeros(3)
    big = 1e9
    assert np.array_equal(oracle.shift_observation(o, z3, z3, big, big), o)
    # shift + clip, exactly at the bound; every other component untouched
    pr, vr = np.array([5.0, -5.0, o[2]]), np.array([0.0, 0.0, -7.0])
    s = oracle.shift_observation(o, pr, vr, 0.3, 1.0)
    assert s[0] == -0.3 and s[1] == 0.3 and s[2] == 0.0
    assert s[12] == min(max(o[12], -1.0), 1.0) and s[14] == 1.0
    keep = np.r_[3:12, 15:len(o)]
    assert np.array_equal(s[keep], o[keep])


def test_tracking_rmse_exact_hover_closed_form():
    """A vehicle that holds its start point (exact hover action, no termination) tracking the
    unit figure-eight from p_ref(0) = (1, 0, z): e^2 = (cos th - 1)^2 + sin^2(2 th)/4, whose mean
    over whole cycles is 3/2 + 1/8, so RMSE = RMSE_xy = sqrt(13/8) (z error 0)."""
    cfg = inputs.config_c4()
    cfg["flags"] &= ~4  # no termination: the full run is scored
    for T, cycles in ((5.5, 1), (3.5, 2), (15.0, 1)):
        n = int(round(T / cfg["dt"])) * cycles
        r, rxy, ok, pos = oracle.track(cfg, None, 0, 0, T, n, z=1.0, trace=True)
        assert ok == n
        assert abs(r - math.sqrt(13 / 8)) < 1e-9 and abs(rxy - r) < 1e-12
        assert np.abs(pos - [1.0, 0.0, 1.0]).max() < 1e-9  # hover: the vehicle does not move


def test_tracking_terminates_on_error_state():
    """With termination on, the hovering vehicle fails when |x error| = 1 - cos(th) first
    exceeds term_pos (|y error| <= 1/2 < 0.6 and the speed error stays < 10 m/s)."""
    cfg = inputs.config_c4()
    T = 5.5
    n = int(round(T / cfg["dt"]))
    _, _, ok, _ = oracle.track(cfg, None, 0, 0, T, n)
    th = math.acos(1.0 - cfg["term_pos"])
    k_fail = math.floor(th * n / (2 * math.pi)) + 1  # first k with 1 - cos(2 pi k / n) > term_pos
    assert ok == k_fail - 1
