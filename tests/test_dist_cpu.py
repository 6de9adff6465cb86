"""Multi-process (gloo, world_size 2) tests of the sharding + statistics all-reduce logic that
bench.py uses on N GPUs (-m "not gpu").  Each rank runs the FP64 oracle on its env-id shard;
the all-reduced statistics must equal a single-process run over all envs, and per-env results
must not depend on the sharding (RNG keyed by global env id, Q20)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
import oracle
from paper_2311_13081_b200 import dist as l2fdist

N_PER, T = 48, 40


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, r, lr = l2fdist.world_info()
    assert (w, r, lr) == (world, rank, rank)
    cfg = inputs.config_c5()
    cfg["curriculum"]["interval"] = 10
    if mode == "weak":
        off, n = l2fdist.shard(rank, world, N_PER)
    else:
        off, n = l2fdist.shard_total(rank, world, 2 * N_PER + 1)
    ids = np.arange(off, off + n, dtype=np.uint64)
    E = oracle.reset_many(cfg, ids, 0)
    st, _ = oracle.rollout(cfg, E, ids, 0, T, oracle.MODE_RANDOM)
    stats = torch.tensor(st, dtype=torch.float64)
    l2fdist.allreduce_stats(stats)
    tmax = l2fdist.max_over_ranks(float(rank + 1), "cpu")
    out_q.put((rank, stats.numpy(), E["s"].copy(), ids, tmax))
    dist.barrier()
    dist.destroy_process_group()


def _run(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


@pytest.mark.parametrize("mode", ["weak", "strong"])
def test_sharded_stats_allreduce_equals_single_run(mode):
    res = _run(mode)
    cfg = inputs.config_c5()
    cfg["curriculum"]["interval"] = 10
    total = 2 * N_PER if mode == "weak" else 2 * N_PER + 1
    ids = np.arange(total, dtype=np.uint64)
    E = oracle.reset_many(cfg, ids, 0)
    st, _ = oracle.rollout(cfg, E, ids, 0, T, oracle.MODE_RANDOM)
    for r in res:
        assert np.allclose(r[1], st, rtol=1e-12, atol=1e-9)   # every rank sees the global SUM
        assert np.array_equal(r[1][[0, 1, 2, 3, 4, 7]], st[[0, 1, 2, 3, 4, 7]])
        assert r[4] == 2.0                                      # max over ranks
    # per-env results are independent of the sharding (global env ids)
    s_cat = np.concatenate([r[2] for r in res])
    assert np.array_equal(np.concatenate([r[3] for r in res]), ids)
    assert np.array_equal(s_cat, E["s"])


def test_shard_arithmetic():
    assert l2fdist.shard(3, 8, 1 << 21) == (3 << 21, 1 << 21)
    parts = [l2fdist.shard_total(r, 3, 10) for r in range(3)]
    assert parts == [(0, 3), (3, 3), (6, 4)]
    with pytest.raises(ValueError):
        l2fdist.shard(2, 2, 5)
