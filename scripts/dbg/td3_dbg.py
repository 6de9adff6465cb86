import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import oracle
import paper_2311_13081_b200 as pkg
from test_gpu_td3 import init_block, make_batch
for I, B in ((146, 256), (34, 100)):
    A = 2
    for hyper in ({"lr_actor": 0.0, "lr_critic": 0.0}, {}):
        td3 = pkg.TD3(A, I, B, hyper=hyper)
        blocks = [init_block(td3, a) for a in range(A)]
        td3.params.copy_(torch.as_tensor(np.stack(blocks)))
        bt = make_batch(A, B, I, 100)
        losses = td3.update({k: torch.as_tensor(v) for k, v in bt.items()}, update_actor=True).cpu().numpy()
        gg = {k: v.cpu().numpy().copy() for k, v in td3.grads().items()}
        for a in range(A):
            lo, go = oracle.td3_update(blocks[a].astype(np.float64), I, {k: v[a].astype(np.float64) for k, v in bt.items()},
                                       td3.hyper, update_actor=True, want_grads=True)
            nc, na = td3.nc, td3.na
            errs = {}
            for name, sl in (("q1", slice(0, nc)), ("q2", slice(nc, 2 * nc)), ("actor", slice(2 * nc, 2 * nc + na))):
                want = go[sl]
                errs[name] = float(np.abs(gg[name][a] - want).max() / np.abs(want).max())
            # segments of the actor gradient
            o = 0
            seg = {}
            for nm, n in (("W1", 64 * I), ("b1", 64), ("W2", 4096), ("b2", 64), ("W3", 256), ("b3", 4)):
                w = go[2 * nc + o:2 * nc + o + n]; g = gg["actor"][a][o:o + n]
                seg[nm] = float(np.abs(g - w).max() / (np.abs(w).max() + 1e-30)); o += n
            print(I, B, "lr0" if hyper else "lr", a, "loss rel", np.abs(losses[a] - lo) / np.abs(lo), errs, seg)
# determinism
td3 = pkg.TD3(2, 146, 256)
blocks = np.stack([init_block(td3, a) for a in range(2)])
bt = {k: torch.as_tensor(v) for k, v in make_batch(2, 256, 146, 100).items()}
outs = []
for rep in range(3):
    td3.params.copy_(torch.as_tensor(blocks))
    l = td3.update(bt, update_actor=True).cpu().numpy().copy()
    outs.append((l, td3.params.cpu().numpy().copy(), {k: v.cpu().numpy().copy() for k, v in td3.grads().items()}))
for rep in (1, 2):
    print("rep", rep, "losses equal", outs[0][0] == outs[rep][0], "params equal", np.array_equal(outs[0][1], outs[rep][1]),
          {k: np.array_equal(outs[0][2][k], outs[rep][2][k]) for k in outs[0][2]})
