"""Pins of the oracle's TD3 update (Q32-Q35), -m "not gpu".

Each check is against something other than the oracle's own formulas: central finite
differences of the losses it reports, the special cases the algorithm fixes (done -> y = r,
tau = 1 hard copy / tau = 0 no change, a critic blind to the action gives no actor
gradient), and Adam's closed-form first step."""
import numpy as np
import pytest

import oracle

IN = 18 + 4 * 4  # a small actor input (N_H = 4)


def make_block(seed=0, in_dim=IN):
    g = np.random.default_rng(seed)
    na, nc = oracle.net_size(in_dim, 64, 4), oracle.net_size(32, 64, 1)
    P = np.zeros(oracle.td3_block_size(in_dim))

    def net(n_in, n_out):
        parts = []
        for (o, i) in ((64, n_in), (64, 64), (n_out, 64)):
            b = 1.0 / np.sqrt(i)
            parts += [g.uniform(-b, b, o * i), g.uniform(-b, b, o)]
        return np.concatenate(parts)

    a, c1, c2 = net(in_dim, 4), net(32, 1), net(32, 1)
    P[:na] = a
    P[na:2 * na] = net(in_dim, 4)  # targets differ from the online nets
    P[2 * na:2 * na + nc] = c1
    P[2 * na + nc:2 * na + 2 * nc] = c2
    P[2 * na + 2 * nc:2 * na + 3 * nc] = net(32, 1)
    P[2 * na + 3 * nc:2 * na + 4 * nc] = net(32, 1)
    return P


def make_batch(B=32, seed=1, in_dim=IN):
    g = np.random.default_rng(seed)
    return {"o_a": g.normal(0, 0.5, (B, in_dim)), "o_c": g.normal(0, 0.5, (B, 28)),
            "a": g.uniform(-1, 1, (B, 4)), "r": g.normal(-1, 1, B), "o_a2": g.normal(0, 0.5, (B, in_dim)),
            "o_c2": g.normal(0, 0.5, (B, 28)), "done": (g.uniform(0, 1, B) < 0.2).astype(float),
            "eps": g.normal(0, 1, (B, 4))}


def offsets(in_dim=IN):
    na, nc = oracle.net_size(in_dim, 64, 4), oracle.net_size(32, 64, 1)
    return {"actor": 0, "actor_t": na, "q1": 2 * na, "q2": 2 * na + nc, "q1_t": 2 * na + 2 * nc,
            "q2_t": 2 * na + 3 * nc, "na": na, "nc": nc}


def test_critic_and_actor_gradients_match_finite_differences():
    P0, b = make_block(), make_batch()
    off = offsets()
    frozen = {"lr_actor": 0.0, "lr_critic": 0.0}
    _, g = oracle.td3_update(P0.copy(), IN, b, frozen, want_grads=True)
    rng = np.random.default_rng(5)

    def losses_at(P):
        return oracle.td3_update(P, IN, b, frozen)[0]

    checked = 0
    for which, li, base, gbase, n in (("q1", 0, off["q1"], 0, off["nc"]), ("q2", 1, off["q2"], off["nc"], off["nc"]),
                                      ("actor", 2, off["actor"], 2 * off["nc"], off["na"])):
        for k in rng.choice(n, 12, replace=False):
            h = 1e-6
            Pp, Pm = P0.copy(), P0.copy()
            Pp[base + k] += h
            Pm[base + k] -= h
            fd = (losses_at(Pp)[li] - losses_at(Pm)[li]) / (2 * h)
            an = g[gbase + k]
            assert abs(fd - an) <= 1e-6 + 1e-5 * abs(an), (which, k, fd, an)
            checked += 1
    assert checked == 36


def test_terminal_transition_target_is_the_reward():
    """done = 1: y = r exactly, so a critic that outputs 0 (all weights 0) has loss mean(r^2)."""
    P, b = make_block(), make_batch()
    off = offsets()
    b["done"][:] = 1.0
    for q in ("q1", "q2"):
        P[off[q]:off[q] + off["nc"]] = 0.0
    losses, _ = oracle.td3_update(P, IN, b, {"lr_critic": 0.0, "lr_actor": 0.0})
    assert np.isclose(losses[0], np.mean(b["r"] ** 2), rtol=1e-14)
    assert np.isclose(losses[1], np.mean(b["r"] ** 2), rtol=1e-14)
    # gamma = 0 gives the same target whatever done is
    b["done"][:] = 0.0
    losses, _ = oracle.td3_update(P, IN, b, {"gamma": 0.0, "lr_critic": 0.0, "lr_actor": 0.0})
    assert np.isclose(losses[0], np.mean(b["r"] ** 2), rtol=1e-14)


def test_polyak_tau_one_copies_tau_zero_keeps():
    off = offsets()
    P, b = make_block(), make_batch()
    oracle.td3_update(P, IN, b, {"tau": 1.0})
    assert np.array_equal(P[off["actor_t"]:off["actor_t"] + off["na"]], P[:off["na"]])
    assert np.array_equal(P[off["q1_t"]:off["q1_t"] + off["nc"]], P[off["q1"]:off["q1"] + off["nc"]])
    P2, P0 = make_block(), make_block()
    oracle.td3_update(P2, IN, b, {"tau": 0.0})
    assert np.array_equal(P2[off["actor_t"]:off["actor_t"] + off["na"]], P0[off["actor_t"]:off["actor_t"] + off["na"]])
    # no actor update on a non-delayed step: actor and targets untouched, critics moved
    P3 = make_block()
    oracle.td3_update(P3, IN, b, update_actor=False)
    assert np.array_equal(P3[:2 * off["na"]], P0[:2 * off["na"]])
    assert not np.array_equal(P3[off["q1"]:off["q1"] + off["nc"]], P0[off["q1"]:off["q1"] + off["nc"]])


def test_adam_first_step_closed_form():
    """t = 1 from zero moments: the step is -lr g / (|g| + eps) (bias corrections cancel)."""
    off = offsets()
    P0, b = make_block(), make_batch()
    P = P0.copy()
    lr = 1e-3
    _, g = oracle.td3_update(P, IN, b, {"lr_critic": lr, "lr_actor": lr}, want_grads=True)
    gq1 = g[:off["nc"]]
    d = P[off["q1"]:off["q1"] + off["nc"]] - P0[off["q1"]:off["q1"] + off["nc"]]
    assert np.allclose(d, -lr * gq1 / (np.abs(gq1) + 1e-8), rtol=1e-9, atol=1e-15)
    ga = g[2 * off["nc"]:]
    d = P[:off["na"]] - P0[:off["na"]]
    assert np.allclose(d, -lr * ga / (np.abs(ga) + 1e-8), rtol=1e-9, atol=1e-15)


def test_critic_blind_to_the_action_gives_no_actor_gradient():
    off = offsets()
    P, b = make_block(), make_batch()
    W1 = P[off["q1"]:off["q1"] + 64 * 32].reshape(64, 32)
    W1[:, 28:] = 0.0  # Q1 ignores the action inputs
    _, g = oracle.td3_update(P, IN, b, {"lr_critic": 0.0}, want_grads=True)
    assert np.all(g[2 * off["nc"]:] == 0.0)
