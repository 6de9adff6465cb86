"""GPU <-> oracle parity of the batched TD3 update, l2f_td3_update (DESIGN.md
Q32-Q35).  The GPU runs FP32, the oracle FP64 on the same (FP32-representable) inputs.

Compared: losses, raw gradients (before Adam; max error <= 1e-4 of the largest entry), and the
updated parameters.  Adam divides by sqrt(v) + eps, so a gradient entry within FP32 noise of
zero can legitimately move its parameter by anything in [-lr, lr]; the updated parameters are
therefore required to stay within Adam's step bound of the oracle everywhere and to agree to
1e-3 lr for the median entry."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2311_13081_b200 as p
    p.lib()
    return p


def init_block(td3, seed):
    """Online nets U(+-1/sqrt(fan_in)), targets different nets, zero moments; FP32 values."""
    g = np.random.default_rng(seed)
    o = td3.offsets()

    def net(n_in, n_out):
        parts = []
        for (m, i) in ((64, n_in), (64, 64), (n_out, 64)):
            b = 1.0 / np.sqrt(i)
            parts += [g.uniform(-b, b, m * i), g.uniform(-b, b, m)]
        return np.concatenate(parts)

    P = np.zeros(td3.block)
    P[o["actor"]:o["actor"] + td3.na] = net(td3.in_dim, 4)
    P[o["actor_t"]:o["actor_t"] + td3.na] = net(td3.in_dim, 4)
    for k in ("q1", "q2", "q1_t", "q2_t"):
        P[o[k]:o[k] + td3.nc] = net(32, 1)
    return P.astype(np.float32)


def make_batch(A, B, I, seed):
    g = np.random.default_rng(seed)
    f = lambda *s: g.normal(0, 0.5, s).astype(np.float32)  # noqa: E731
    return {"o_a": f(A, B, I), "o_c": f(A, B, 28), "a": g.uniform(-1, 1, (A, B, 4)).astype(np.float32),
            "r": g.normal(-1, 1, (A, B)).astype(np.float32), "o_a2": f(A, B, I), "o_c2": f(A, B, 28),
            "done": (g.uniform(0, 1, (A, B)) < 0.2).astype(np.float32), "eps": g.normal(0, 1, (A, B, 4)).astype(np.float32)}


def run_both(pkg, A, B, I, steps, hyper=None, seed=0):
    td3 = pkg.TD3(A, I, B, hyper=hyper)
    blocks = [init_block(td3, seed + a) for a in range(A)]
    td3.params.copy_(torch.as_tensor(np.stack(blocks)))
    P_or = [b.astype(np.float64) for b in blocks]
    res = []
    for k, upd in enumerate(steps):
        bt = make_batch(A, B, I, 100 + k)
        losses = td3.update({kk: torch.as_tensor(v) for kk, v in bt.items()}, update_actor=upd).cpu().numpy()
        gg = {kk: v.cpu().numpy().copy() for kk, v in td3.grads().items()}
        ref = []
        for a in range(A):
            ba = {kk: v[a].astype(np.float64) for kk, v in bt.items()}
            lo, go = oracle.td3_update(P_or[a], I, ba, td3.hyper, t_critic=td3.t_critic, t_actor=max(td3.t_actor, 1),
                                       update_actor=upd, want_grads=True)
            ref.append((lo, go))
        res.append((losses, gg, ref))
    return td3, P_or, res


@pytest.mark.parametrize("I,B", [(146, 256), (34, 100)])
def test_td3_update_matches_oracle(pkg, I, B):
    A = 3
    td3, P_or, res = run_both(pkg, A, B, I, [True, False, True])
    nc, na = td3.nc, td3.na
    for (losses, gg, ref) in res:
        for a in range(A):
            lo, go = ref[a]
            assert np.allclose(losses[a], lo, rtol=2e-4, atol=1e-6), (a, losses[a], lo)
            for name, sl, n in (("q1", slice(0, nc), nc), ("q2", slice(nc, 2 * nc), nc), ("actor", slice(2 * nc, 2 * nc + na), na)):
                if name == "actor" and lo[2] == 0.0:
                    continue
                want = go[sl]
                scale = np.abs(want).max()
                assert np.abs(gg[name][a] - want).max() <= 1e-4 * scale + 1e-7, (name, a)
    # parameters after the three updates
    P_gpu = td3.params.cpu().numpy().astype(np.float64)
    lr = td3.hyper["lr_critic"]
    for a in range(A):
        d = np.abs(P_gpu[a] - P_or[a])
        assert d.max() <= 3 * lr + 1e-6  # never more than Adam's step bound apart
        assert np.median(d) <= 1e-3 * lr + 1e-7  # and almost everywhere FP32-close


def test_td3_special_cases(pkg):
    """tau = 1 copies the online nets into the targets exactly; done = 1 with zero critics
    gives the critic loss mean(r^2); no actor step leaves actor and targets untouched."""
    A, B, I = 2, 64, 34
    td3 = pkg.TD3(A, I, B, hyper={"tau": 1.0})
    blocks = [init_block(td3, 7 + a) for a in range(A)]
    o = td3.offsets()
    for b in blocks:
        b[o["q1"]:o["q1"] + td3.nc] = 0.0
        b[o["q2"]:o["q2"] + td3.nc] = 0.0
    td3.params.copy_(torch.as_tensor(np.stack(blocks)))
    bt = make_batch(A, B, I, 5)
    bt["done"][:] = 1.0
    before = td3.params.clone()
    losses = td3.update({k: torch.as_tensor(v) for k, v in bt.items()}, update_actor=False).cpu().numpy()
    for a in range(A):
        assert np.isclose(losses[a, 0], np.mean(bt["r"][a].astype(np.float64) ** 2), rtol=1e-5)
        assert losses[a, 2] == 0.0
    P = td3.params
    assert torch.equal(P[:, :2 * td3.na], before[:, :2 * td3.na])  # actor + actor' untouched
    td3.update({k: torch.as_tensor(v) for k, v in bt.items()}, update_actor=True)
    P = td3.params
    assert torch.equal(P[:, o["actor_t"]:o["actor_t"] + td3.na], P[:, :td3.na])
    assert torch.equal(P[:, o["q1_t"]:o["q1_t"] + td3.nc], P[:, o["q1"]:o["q1"] + td3.nc])
    assert torch.equal(P[:, o["q2_t"]:o["q2_t"] + td3.nc], P[:, o["q2"]:o["q2"] + td3.nc])


def test_td3_actor_exports_to_the_rollout(pkg):
    """The learner's actor (fp16-rounded) drives the tcgen05 policy path."""
    import inputs
    td3 = pkg.TD3(1, 146, 32)
    td3.params.copy_(torch.as_tensor(init_block(td3, 3))[None])
    W = td3.actor_policy_weights(0)
    env = pkg.Env(inputs.config_c4(), 256)
    env.reset()
    env.rollout(5, policy=pkg.Policy(W))
    assert torch.isfinite(env.state).all()


@pytest.mark.parametrize("A,B,I", [(1, 1, 18), (5, 33, 18), (2, 256, 146), (2, 77, 35), (1, 256, 156)])
def test_td3_edge_shapes_match_oracle(pkg, A, B, I):
    """Single-sample batch, N_H = 0 actor input (in_dim 18), ragged batch, full batch, an odd
    in_dim (4-byte staging path), the largest supported in_dim (two staged column parts)."""
    td3, P_or, res = run_both(pkg, A, B, I, [True], seed=11)
    losses, gg, ref = res[0]
    for a in range(A):
        assert np.allclose(losses[a], ref[a][0], rtol=2e-4, atol=1e-6)
        go = ref[a][1]
        scale = np.abs(go[:td3.nc]).max()
        assert np.abs(gg["q1"][a] - go[:td3.nc]).max() <= 1e-4 * scale + 1e-7


def test_td3_invalid_arguments(pkg):
    with pytest.raises(Exception):
        pkg.TD3(1, 146, 0)
    with pytest.raises(Exception):
        pkg.TD3(1, 146, 257)
    with pytest.raises(Exception):
        pkg.TD3(1, 157, 64)  # beyond the kernel's shared-memory plan
    td3 = pkg.TD3(2, 34, 16)
    bt = {k: torch.as_tensor(v) for k, v in make_batch(2, 16, 34, 1).items()}
    bt["o_c"] = bt["o_c"][:, :8]  # wrong batch size
    with pytest.raises(ValueError):
        td3.update(bt, update_actor=True)


def test_td3_update_is_deterministic(pkg):
    """The partial gradients are summed in a fixed order: two learners fed the same state and
    batch end bitwise equal (losses, gradients, parameters)."""
    A, B, I = 3, 256, 146
    bt = {k: torch.as_tensor(v) for k, v in make_batch(A, B, I, 9).items()}
    res = []
    for _ in range(2):
        td3 = pkg.TD3(A, I, B)
        td3.params.copy_(torch.as_tensor(np.stack([init_block(td3, 40 + a) for a in range(A)])))
        l1 = td3.update(bt, update_actor=False).clone()
        l2 = td3.update(bt, update_actor=True).clone()
        res.append((l1, l2, td3.params.clone(), {k: v.clone() for k, v in td3.grads().items()}))
    (a1, a2, ap, ag), (b1, b2, bp, bg) = res
    assert torch.equal(a1, b1) and torch.equal(a2, b2) and torch.equal(ap, bp)
    assert all(torch.equal(ag[k], bg[k]) for k in ag)


def test_td3_export_actor_on_device_matches_host_rounding(pkg):
    """l2f_td3_export_actor == fp16 RNE of the actor block (numpy), and the exported policy
    drives policy_forward identically to the host-converted one."""
    td3 = pkg.TD3(3, 146, 32)
    td3.params.copy_(torch.as_tensor(np.stack([init_block(td3, 20 + a) for a in range(3)])))
    pol_dev = td3.actor_policy(agent=2)
    W = td3.actor_policy_weights(2)
    host = np.concatenate([W[k].ravel() for k in ("W1", "b1", "W2", "b2", "W3", "b3")])
    dev = pol_dev.t["buf"].cpu().numpy().view(np.uint16)
    assert np.array_equal(dev, host)
    obs = torch.randn(1000, 146, device="cuda") * 0.3
    a1 = pkg.policy_forward(pol_dev, obs)
    a2 = pkg.policy_forward(pkg.Policy(W), obs)
    assert torch.equal(a1, a2)


def test_td3_bench_configuration_sampled(pkg):
    """The bench's configuration (148 agents x batch 256 x in_dim 146, one CTA per SM): three
    sampled agents' losses and critic/actor gradients vs the oracle."""
    A, B, I = 148, 256, 146
    td3 = pkg.TD3(A, I, B)
    blocks = np.stack([init_block(td3, 50 + (a % 7)) for a in range(A)])
    td3.params.copy_(torch.as_tensor(blocks))
    bt = make_batch(A, B, I, 77)
    losses = td3.update({k: torch.as_tensor(v) for k, v in bt.items()}, update_actor=True).cpu().numpy()
    gg = {k: v.cpu().numpy() for k, v in td3.grads().items()}
    for a in (0, 73, 147):
        P = blocks[a].astype(np.float64)
        lo, go = oracle.td3_update(P, I, {k: v[a].astype(np.float64) for k, v in bt.items()}, td3.hyper,
                                   update_actor=True, want_grads=True)
        assert np.allclose(losses[a], lo, rtol=2e-4, atol=1e-6)
        nc = td3.nc
        for name, ref in (("q1", go[:nc]), ("q2", go[nc:2 * nc]), ("actor", go[2 * nc:])):
            assert np.abs(gg[name][a] - ref).max() <= 1e-4 * np.abs(ref).max() + 1e-7, (a, name)
