"""GPU <-> oracle parity on the method's degenerate cases (-m gpu):

* divergence: a non-finite state (NaN or +-Inf in any block) ends the episode as
  DIVERGED | TERMINATED with reward 0 (Q26), through l2f_step and
  through the fused rollouts;
* exact thresholds: ||p||_inf = 0.6, ||v|| = 10, ||w|| = 35 exactly are NOT terminal (strict
  >), one fp32 ulp above is (Q14).  The states are built so that the step keeps
  the thresholded component exactly (level attitude, rotors off or at hover, no disturbance),
  so both sides see the value itself, not a rounded neighbour.
Every flag is compared bit for bit with the oracle; no Q22 exclusion applies here because the
margins are exactly 0 or one ulp by construction."""
import numpy as np
import pytest
import torch

import inputs
import oracle
from gpu_helpers import load_snapshot, snapshot, to_oracle

pytestmark = pytest.mark.gpu

P = inputs.CRAZYFLIE
HOVER = float(np.sqrt(P["mass"] * P["gravity"] / (4 * P["thrust_c"][2])))
A_HOVER = 2 * HOVER / P["rpm_max"] - 1  # exact normalised hover action for rpm_min = 0


@pytest.fixture(scope="module")
def pkg():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2311_13081_b200 as p
    p.lib()
    return p


def f32(x):
    return float(np.float32(x))


def up(x):
    return float(np.nextafter(np.float32(x), np.float32(np.inf)))


def level_states(rows):
    """rows: list of dicts {p, v, w, rotors} -> SoA state [17][n], level attitude.  rotors
    "off": speed 0 held by the action -1 (every thrust and torque exactly 0, a free fall);
    "hover": the hover speed held by the hover action (residual accelerations ~1e-8, far
    below one ulp of the thresholded components)."""
    n = len(rows)
    s = np.zeros((17, n))
    s[3] = 1.0
    for i, r in enumerate(rows):
        s[0:3, i] = r.get("p", (0, 0, 0))
        s[7:10, i] = r.get("v", (0, 0, 0))
        s[10:13, i] = r.get("w", (0, 0, 0))
        s[13:17, i] = HOVER if r.get("rotors", "hover") == "hover" else 0.0
    return s


def case_actions(rows, n):
    a = np.full((4, n), np.float32(A_HOVER))
    for i, r in enumerate(rows):
        if r.get("rotors", "hover") == "off":
            a[:, i] = -1.0
    return a


# The position bound of these cases: 0.6 (Q14) has no fp32 representation -- the kernel
# compares against fp32(0.6) = 0.6000000238, the oracle against 0.6 -- so "exactly at the
# bound" is tested at 0.625, a bound both sides hold exactly (Q37).  |v| = 10 and
# |w| = 35 (squared: 100, 1225) are exact in both precisions.
POS = 0.625

# (case, terminated?)
CASES = [
    ({"p": (POS, 0, 0), "rotors": "off"}, False),     # exactly at the position bound
    ({"p": (up(POS), 0, 0), "rotors": "off"}, True),  # one ulp above
    ({"p": (0, -POS, 0), "rotors": "off"}, False),    # negative side, exactly
    ({"p": (0, 0, -up(POS)), "rotors": "off"}, True), # beyond, and falling
    ({"v": (10.0, 0, 0)}, False),                        # |v| = 10 exactly
    ({"v": (up(10.0), 0, 0)}, True),
    ({"w": (35.0, 0, 0), "rotors": "off"}, False),       # |w| = 35 about a principal axis
    ({"w": (0, 0, up(35.0)), "rotors": "off"}, True),
    ({"v": (6.0, 8.0, 0)}, False),                       # |v|^2 = 100 exactly from two components
    ({}, False),                                         # hover at the origin
]
ROWS = [c for c, _ in CASES]


def edge_config(flags):
    cfg = inputs.base_config(flags=flags, seed=17)
    cfg["term_pos"] = POS
    return cfg


def _edge_env(pkg, cfg, rows, extra_states=None):
    n = len(rows) + (extra_states.shape[1] if extra_states is not None else 0)
    env = pkg.Env(cfg, n)
    env.reset()
    s = level_states(rows)
    if extra_states is not None:
        s = np.concatenate([s, extra_states], axis=1)
    snap = {"state": s, "dist": np.zeros((6, n)), "dr": np.ones((5, n)),
            "hist": np.full((cfg["n_hist"], 4, n), A_HOVER), "hist_t0": np.full(n, -(1 << 30), dtype=np.int32),
            "hist_fill": np.full((4, n), A_HOVER), "ep_step": np.full(n, 7, dtype=np.int32),
            "ep_return": np.zeros(n)}
    load_snapshot(env, snap)
    return env, snapshot(env), n


def _divergent_states():
    """Non-finite states (non-finite on both sides; a finite fp32 overflow is divergence only
    in FP32 and is not compared)."""
    s = level_states([{}] * 4)
    s[7, 0] = np.nan            # NaN velocity
    s[0, 1] = np.inf            # +Inf position
    s[12, 2] = -np.inf          # -Inf body rate
    s[13, 3] = np.nan           # NaN rotor speed
    return s


N_DIV = 4


@pytest.mark.parametrize("auto_reset", [False, True])
def test_step_thresholds_and_divergence_match_oracle(pkg, auto_reset):
    flags = inputs.TERMINATION | (inputs.AUTO_RESET if auto_reset else 0)
    cfg = edge_config(flags)
    env, snap, n = _edge_env(pkg, cfg, ROWS, _divergent_states())
    t = 50
    env.t = t
    a = case_actions(ROWS, n)
    acts = torch.tensor(a, dtype=torch.float32, device="cuda")
    out = env.make_out(final_state=True)
    env.step(acts, out)
    flg = out["flags"].cpu().numpy().astype(int)
    rew = out["reward"].cpu().numpy()
    fin = out["final_state"].cpu().numpy()
    E = to_oracle(snap, np.arange(n), t, cfg["n_hist"])
    exp_term = [term for _, term in CASES] + [True] * N_DIV
    for i in range(n):
        so = oracle.env_step(cfg, E[i:i + 1], i, t, a[:, i].astype(np.float32).astype(np.float64))
        assert flg[i] == so.flags, (i, flg[i], so.flags)
        assert bool(so.flags & oracle.FLAG_TERMINATED) == exp_term[i], (i, so.flags)
        if i < len(ROWS):
            # the thresholded component is carried exactly through the step on both sides
            assert not so.flags & oracle.FLAG_DIVERGED
            for k in (0, 1, 2, 7, 8, 9, 10, 11, 12):
                if snap["state"][k, i] != 0.0 and k not in (2, 9):  # z / v_z move under the thrust residual
                    assert fin[k, i] == snap["state"][k, i] == so.final_s[k], (i, k)
        else:
            assert so.flags & oracle.FLAG_DIVERGED and so.flags & oracle.FLAG_TERMINATED, (i, so.flags)
            assert rew[i] == 0.0 and so.reward == 0.0, (i, rew[i])
            assert bool(flg[i] & oracle.FLAG_RESET) == auto_reset
    if auto_reset:  # the diverged envs restart from finite reset states
        after = snapshot(env)
        assert np.all(np.isfinite(after["state"][:, len(ROWS):]))
    st = env.episode_stats().cpu().numpy()
    assert st[3] == N_DIV and st[1] == N_DIV + sum(term for _, term in CASES)  # diverged, terminated


def test_rollout_divergence_and_threshold(pkg):
    """The same cases through the fused open-loop rollout (one step with recorded actions):
    flags and reward 0 on divergence, identical to l2f_step."""
    cfg = edge_config(inputs.TERMINATION | inputs.AUTO_RESET)
    env, snap, n = _edge_env(pkg, cfg, ROWS, _divergent_states())
    env.t = 50
    acts = torch.tensor(case_actions(ROWS, n)[None], dtype=torch.float32, device="cuda")
    tr = env.rollout(1, actions=acts, trace_ids=torch.arange(n)).cpu().numpy()
    env2, _, _ = _edge_env(pkg, cfg, ROWS, _divergent_states())
    env2.t = 50
    out = env2.make_out()
    env2.step(acts[0].contiguous(), out)
    assert np.array_equal(tr[0, :, 26].astype(int), out["flags"].cpu().numpy().astype(int))
    assert np.array_equal(tr[0, :, 25], out["reward"].cpu().numpy())
    assert np.all(tr[0, len(ROWS):, 25] == 0.0)


def test_mlp_rollout_divergence(pkg):
    """A non-finite state inside the fused MLP rollout: DIVERGED | TERMINATED, reward 0, the
    env restarts finite and the rest of the batch is unaffected (bitwise equal to a run
    without the poisoned envs)."""
    cfg = inputs.config_c4(seed=23)
    n = 3 * 128
    W = inputs.policy_weights(146, 64, seed=7, out_bias=inputs.hover_policy_bias())
    pol = pkg.Policy(W)
    env = pkg.Env(cfg, n)
    env.reset()
    ref = pkg.Env(cfg, n)
    ref.reset()
    bad = [5, 200, 383]
    s = env.state.cpu().numpy()
    s[7, 5] = np.nan
    s[0, 200] = np.inf
    s[12, 383] = -np.inf
    env.set_logical("state", s)
    tr = env.rollout(3, policy=pol, trace_ids=torch.as_tensor(bad)).cpu().numpy()
    ref.rollout(3, policy=pol)
    fl = tr[0, :, 26].astype(int)
    assert np.all(fl & oracle.FLAG_DIVERGED) and np.all(fl & oracle.FLAG_TERMINATED), fl
    assert np.all(tr[0, :, 25] == 0.0)
    assert np.all(np.isfinite(tr[1:, :, :17]))
    a, b = snapshot(env), snapshot(ref)
    keep = np.setdiff1d(np.arange(n), bad)
    for k in ("state", "dist", "ep_step", "ep_return"):
        assert np.array_equal(a[k][..., keep], b[k][..., keep]), k
