"""bench.py's GPU arm prints the contract's JSON line (-m gpu): metric/config shared with the
reference arm, whole-job value, roofline with a measured fraction, end-to-end number with the
bytes it moved, launch count, sampled clocks.  A short run (1 timed step of the real 2^21-env
x 1000-step workload, secondary modes and CPU baseline off)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    sys.path.insert(0, ROOT)
    import bench
    r = subprocess.run([sys.executable, "bench.py", "--steps", "1", "--warmup", "3", "--no-secondary",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["metric"] == bench.METRIC and d["unit"] == "env-steps/s" and d["higher_is_better"] is True
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3 and d["scaling"] == "weak"
    assert d["config"] == bench.main_config(bench.ENVS_PER_GPU, bench.T_ROLLOUT, "mlp", 1)
    n, T = bench.ENVS_PER_GPU, bench.T_ROLLOUT
    assert abs(d["value"] - n * T / (d["ms_per_step"] * 1e-3)) <= 1e-6 * d["value"]
    rf = d["roofline"]
    assert rf["bound"] == "alu" and 0.0 < rf["frac"] < 1.0 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e = d["e2e"]
    assert e["unit"] == "env-steps/s" and e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 1
    assert d["clocks"]["sm_mhz"] > 0 and isinstance(d["clocks"]["reasons"], list)


def _run_bench(args, extra_env):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(extra_env)
    r = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_two_ranks_reduce_stats_like_one_rank():
    """The multi-rank bench path end to end -- self-launch under torch.distributed.run, shard
    offsets, barriers, max-over-ranks timing, the statistics all-reduce (a15) -- with 2 ranks on
    the test box's one GPU over gloo (L2F_DIST_BACKEND; the ranks' kernels never wait on one
    another).  The all-reduced episode statistics of 2 x 4096 envs equal a 1-rank run over the
    same 8192 global env ids."""
    common = ["--steps", "1", "--warmup", "3", "--no-secondary", "--no-cpu-baseline", "--T", "60"]
    d2 = _run_bench(["--gpus", "2", "--envs-per-gpu", "4096"] + common, {"L2F_DIST_BACKEND": "gloo"})
    d1 = _run_bench(["--gpus", "1", "--envs-per-gpu", "8192"] + common, {})
    assert d2["n_gpus"] == 2 and d2["value"] > 0 and d2["config"]["parallelism"] == "env-shard x2"
    s1, s2 = d1["episode_stats"], d2["episode_stats"]
    assert s2["episodes"] == s1["episodes"] > 0
    assert abs(s2["mean_len"] - s1["mean_len"]) <= 1e-12 * s1["mean_len"]
    assert abs(s2["mean_return"] - s1["mean_return"]) <= 1e-9 * abs(s1["mean_return"])
