#!/usr/bin/env python3
"""Benchmark of the batched quadrotor env hot path (arXiv 2311.13081) on B200.

  python bench.py --gpus N --steps K --warmup W [--impl reference]
  (N > 1 without a torchrun environment: bench.py re-launches itself as
   python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 ...
   one rank per GPU; launched under torchrun it runs as the given rank)

One bench "step" = one pass of the whole hot path over the
per-GPU batch: l2f_rollout of T = 1000 env-steps with the actor MLP on tensor cores, noise,
reward + curriculum, termination, auto-reset and DR-free C5 physics, then the episode-stat
reduction and (N > 1) its NCCL all-reduce.  Workload (BASELINE configs[4], per GPU shard):
2^21 envs per GPU x 1000 steps; at N = 8 this is exactly the 2^24-env C5 config; weak scaling.

Prints ONE JSON line (rank 0).  Secondary measurements ride along under "modes": the C3
single-step API against the HBM roofline (and its host-buffer e2e), reward recalculation over
a replay buffer (f2, HBM roofline), the open-loop dynamics-only mode next to the paper's
figure, the C5 env step without the MLP, Lissajous tracking (f3) and the batched TD3 update
(f4, FP32 roofline).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

T_ROLLOUT = 1000
ENVS_PER_GPU = 1 << 21
METRIC = "env-steps/s (sim flight-s per wall-s) at 1/2/4/8 B200 vs roofline"
DT = 0.01
# Algorithmic work per env-step:
#  HBM bytes of one l2f_step with DR (C3): reads state 68 + action 16 + dist 24 + DR 20 +
#  ep counters 8; writes state 68 + counters 8 + history slot 16 + obs_core 72 + reward 4 + flags 1
STEP_BYTES_DR = 68 + 16 + 24 + 20 + 8 + 68 + 8 + 16 + 72 + 4 + 1
#  tensor-core FLOPs of the actor MLP 146 -> 64 -> 64 -> 4 per env-step
MLP_FLOPS = 2 * (146 * 64 + 64 * 64 + 64 * 4)
#  Scalar (non-tensor) work of one env-step for the ALU (issue) roofline: the method's arithmetic
#  instructions per env-step counted mechanically from the kernel's SASS (scripts/alu_ops.py over
#  the committed ncu --set full capture -> profiles/alu_ops.json).  The
#  round-1 hand table is kept beside it for comparison (it counted packed FFMA2 pairs as two).
ALU_OPS_HAND = {"mlp": 1071, "open_c5": 657, "open_dyn": 532}
SMS = 148


def alu_ops(kind):
    """(method ops per env-step, source) of kernel kind 'mlp' / 'open_c5' / 'open_dyn' / 'step'."""
    try:
        with open(os.path.join(ROOT, "profiles", "alu_ops.json")) as f:
            d = json.load(f)[kind]
        return d["method_ops_per_env_step"], d["source"]
    except Exception:
        return ALU_OPS_HAND[kind], "hand count (DESIGN.md section 5.5; profiles/alu_ops.json missing)"


def traffic(key):
    """DRAM bytes per launch of a kernel from the last committed ncu --set full capture
    (profiles/latest_traffic.json, written by scripts/summarize_profile.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "latest_traffic.json")) as f:
            return json.load(f)[key]["dram_bytes"]
    except Exception:
        return None


def peaks():
    p = {"hbm_gbs": 6551.4, "bf16_tflops": 1653.4, "bf16_tflops_sustained": 1387.6, "sm_max_mhz": 1965.0,
         "source": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained", "sm_max_mhz") if k in m})
        p["source"] = "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    return p


# ----------------------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()  # nvidia-smi takes a moment to start: have it sampling before the region
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.first = len(self.lines)  # samples from here on fall inside the timed region
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        # samples taken inside the region; for a region shorter than the 200 ms sampling period,
        # the sample just before it (the GPU was already warm)
        lines = self.lines[self.first:] or self.lines[-1:]
        for l in lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------------------
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: one rank per GPU")
    return world, rank, local


def self_launch(args):
    """--gpus N > 1 outside torchrun: re-run this command as N ranks of one node under
    torch.distributed.run (rendezvous on 127.0.0.1, a free port) and return its exit code.
    NCCL's init log (NCCL_DEBUG=INFO, INIT subsystem) goes to stderr so the rank count is
    visible without touching the one JSON line on stdout."""
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def cpu_baseline(cfg, policy_w, target_s=15.0, nthreads=None):
    """The oracle as it stands (FP64 C, pthreads over all host cores) on a bounded sample of the
    same workload: n_s envs (ids spread over the GPU's shard) x T_s fused MLP env-steps, with
    n_s sized from a short probe so the sample costs about target_s seconds."""
    import numpy as np

    import oracle

    nthreads = nthreads or os.cpu_count() or 1
    pol = oracle.PolicyHandle(policy_w)
    n_p = nthreads * 4
    ids = np.arange(n_p, dtype=np.uint64) * 997
    E = oracle.reset_many(cfg, ids, 0)
    t0 = time.perf_counter()
    oracle.rollout(cfg, E, ids, 0, 20, oracle.MODE_POLICY, policy=pol, nthreads=nthreads)
    rate = n_p * 20 / max(time.perf_counter() - t0, 1e-6)
    T_s = 250
    n_s = int(max(nthreads, min(1 << 16, target_s * rate / T_s)))
    n_s -= n_s % nthreads if n_s >= nthreads else 0
    ids = (np.arange(n_s, dtype=np.uint64) * ((ENVS_PER_GPU // max(n_s, 1)) or 1)).astype(np.uint64)
    E = oracle.reset_many(cfg, ids, 0)
    t0 = time.perf_counter()
    oracle.rollout(cfg, E, ids, 0, T_s, oracle.MODE_POLICY, policy=pol, nthreads=nthreads)
    el = time.perf_counter() - t0
    v = n_s * T_s / el
    return {"value": v, "unit": "env-steps/s", "cores": nthreads, "kind": "oracle",
            "sample": f"{n_s} envs (ids spread over the 2^21-env shard) x {T_s} fused MLP env-steps of the "
                      f"C5 workload, FP64 C oracle on {nthreads} threads, {el:.1f} s wall"}


def main_config(n, T, mode, world):
    """The workload both arms report (the reference arm times a bounded sample of it)."""
    what = ("fused actor-MLP rollout (146-64-64-4 tcgen05, N_H=32)" if mode == "mlp"
            else "open-loop rollout (Philox random actions, no actor MLP)")
    return {"workload": f"C5 per-GPU shard: 2^21 envs/GPU x 1000 steps {what}, obs/action noise, reward + "
                        "4-stage curriculum, termination, auto-reset, disturbance; NCCL stat all-reduce",
            "envs_per_gpu": n, "steps_per_rollout": T, "mode": mode,
            "l2": "inputs larger than L2: env state+history 1.4 GB per GPU",
            "parallelism": f"env-shard x{world}"}


def reference_arm(args):
    """--impl reference: the oracle (the base contract's reference arm for this tier)."""
    world, rank, local = dist_setup(args)
    if rank != 0:
        return
    import inputs

    cfg = inputs.config_c5()
    W = inputs.policy_weights(18 + 4 * cfg["n_hist"], 64, seed=7, out_bias=inputs.hover_policy_bias())
    target = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    target = float(os.environ.get("L2F_REF_TARGET_S", target))  # (tests: a short sample)
    vals = []
    cb = None
    walls = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        cb = cpu_baseline(cfg, W, target_s=target)
        if k >= args.warmup:
            vals.append(cb["value"])
            walls.append(time.perf_counter() - t0)
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "env-steps/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls),
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": main_config(ENVS_PER_GPU, T_ROLLOUT, "mlp", args.gpus),
            "cpu_baseline": dict(cb, value=v),
            "e2e": {"value": v, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "sim_seconds_per_wall_second": v * DT}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs-per-gpu", type=int, default=ENVS_PER_GPU)
    ap.add_argument("--T", type=int, default=T_ROLLOUT)
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="mlp", choices=["mlp", "open"])  # open: Philox random actions, no MLP
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(args))
    if args.impl == "reference":
        return reference_arm(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import inputs
    import paper_2311_13081_b200 as pkg
    from paper_2311_13081_b200 import dist as l2fdist

    world, rank, local = dist_setup(args)
    # One rank per GPU over NCCL.  L2F_DIST_BACKEND=gloo (tests only) runs the same multi-rank
    # path with host-side collectives, so several ranks can share the one GPU of a test box (the
    # ranks' kernels never wait on one another: the only exchange is the stats all-reduce).
    backend = os.environ.get("L2F_DIST_BACKEND", "nccl")
    gpu = local if backend == "nccl" else local % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if backend == "nccl":
            # NCCL's init log (ranks, devices, transports) on stderr, whoever launched the ranks
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    pk = peaks()
    n = args.envs_per_gpu
    T = args.T
    stream = torch.cuda.current_stream()

    cfg = inputs.config_c5()
    W = inputs.policy_weights(18 + 4 * cfg["n_hist"], 64, seed=7, out_bias=inputs.hover_policy_bias())
    offset, n = l2fdist.shard(rank, world, n)  # weak scaling: rank r owns ids [r n, (r+1) n)
    env = pkg.Env(cfg, n, env_id_offset=offset, device=dev)
    env.reset()
    pol = pkg.Policy(W, device=dev)
    stats_buf = torch.zeros(8, dtype=torch.float64, device=dev)

    def one_step():
        if args.mode == "mlp":
            env.rollout(T, policy=pol)
        else:
            env.rollout(T)  # open loop, Philox random actions
        st = env.episode_stats(reset=True)
        l2fdist.allreduce_stats(st)  # a15: NCCL SUM of the FP64 episode statistics
        stats_buf.add_(st)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        one_step()
    barrier()
    stats_buf.zero_()
    l0 = pkg.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            one_step()
        ev1.record(stream)
        barrier()
    launches = pkg.launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    ms_max = l2fdist.max_over_ranks(ms, dev)
    env_steps = world * n * T * args.steps
    value = env_steps / (ms_max / 1e3)
    stats = stats_buf.cpu().numpy()

    # per-launch time of the dominant kernel (the fused rollout) on its own stream
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    if args.mode == "mlp":
        env.rollout(T, policy=pol)
    else:
        env.rollout(T)
    ev3.record(stream)
    torch.cuda.synchronize()
    k_ms = ev2.elapsed_time(ev3)
    clocks = clk.summary()
    f_clk = (clocks["sm_mhz"] or pk["sm_max_mhz"]) * 1e6
    k_rate = n * T / (k_ms / 1e3)
    alu_peak = SMS * 128 * f_clk / 1e12
    kind = "mlp" if args.mode == "mlp" else "open_c5"
    ops, ops_src = alu_ops(kind)
    roof = {"bound": "alu", "kernel": "rollout_mlp_kernel" if args.mode == "mlp" else "rollout_open_kernel",
            "achieved": ops * k_rate / 1e12, "peak": alu_peak, "unit": "Tops/s",
            "frac": ops * k_rate / 1e12 / alu_peak, "ops_per_env_step": ops, "ops_source": ops_src,
            "frac_round1_hand_count": ALU_OPS_HAND[kind] * k_rate / 1e12 / alu_peak,
            "traffic": traffic(kind),
            "traffic_note": "DRAM read+write bytes of one launch of the same kernel and workload (ncu --set full, "
                            "profiles/latest_traffic.json): state and history move once per env per launch",
            "peak_source": f"148 SMs x 128 lanes x {f_clk / 1e6:.0f} MHz (median SM clock sampled in the timed region)",
            "tensor": {"achieved": MLP_FLOPS * k_rate / 1e12, "peak": pk["bf16_tflops_sustained"],
                       "unit": "TFLOP/s", "frac": MLP_FLOPS * k_rate / 1e12 / pk["bf16_tflops_sustained"],
                       "peak_source": pk["source"] + " bf16 sustained (fp16 dense rate equal)"}}

    # ---- e2e through the public host-buffer API: H2D of the policy (pinned), rollout, D2H stats
    e2e_val, h2d = None, 0
    if args.mode == "mlp":
        e2e_val, h2d = e2e_rollout(args, pkg, torch, l2fdist, env, W, T, n, world, dev, stream, barrier)
    modes = {}
    if not args.no_secondary and rank == 0:
        modes = secondary(pkg, inputs, torch, dev, pk, f_clk)
    cb = None
    if rank == 0 and not args.no_cpu_baseline:
        cb = cpu_baseline(cfg, W)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32+f16mma" if args.mode == "mlp" else "f32", "data": "synthetic",
                "config": main_config(n, T, args.mode, world),
                "sim_seconds_per_wall_second": value * DT,
                "roofline": roof,
                "e2e": {"value": e2e_val, "unit": "env-steps/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": 64,
                        "api": "l2f_rollout_host (pinned host policy in, FP64 stats out)"},
                "gpu_launches": int(launches),
                "clocks": clocks,
                "episode_stats": {"episodes": stats[0], "mean_len": stats[4] / max(stats[0], 1),
                                  "mean_return": stats[5] / max(stats[0], 1)},
                "modes": modes,
                "cpu_baseline": cb,
                "paper_context": {"value": 1.284e9, "unit": "env-steps/s", "hardware": "Quadro T2000 laptop GPU",
                                  "workload": "8192 envs x 1e6 steps, forward dynamics only (P:165)"}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def e2e_rollout(args, pkg, torch, l2fdist, env, W, T, n, world, dev, stream, barrier):
    hpol = pkg.HostPolicy(W)
    h_stats = torch.zeros(8, dtype=torch.float64).pin_memory()
    h2d = sum(int(t.numel()) * 2 for t in hpol.t.values())
    e2e_env = env
    for _ in range(1):
        e2e_env.rollout_host(hpol, T, h_stats)
    barrier()
    t0 = time.perf_counter()
    ev4, ev5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev4.record(stream)
    for _ in range(args.steps):
        e2e_env.rollout_host(hpol, T, h_stats)
        if world > 1:
            l2fdist.allreduce_stats(torch.from_numpy(h_stats.numpy().copy()).to(dev))
    ev5.record(stream)
    barrier()
    e2e_ms = l2fdist.max_over_ranks(ev4.elapsed_time(ev5), dev)
    e2e_val = world * n * T * args.steps / (e2e_ms / 1e3)

    return e2e_val, h2d


def small_configs(pkg, inputs, torch, dev):
    """BASELINE configs[0, 1] (C1: 64 x 500, C2: 4096 x 1000): latency-bound sizes, reported as
    absolute env-steps/s and us per step through (a) the open-loop fused rollout (one launch) and
    (b) l2f_step captured T times in one CUDA graph (the graph replays the captured counters)."""
    out = {}
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, cfg, n, T, acts in (
            ("C1", inputs.config_c1(), 64, 500, inputs.actions_uniform(500, 64, seed=11)),
            ("C2", inputs.config_c2(), 4096, 1000, inputs.actions_near_hover(1000, 4096, seed=12))):
        a = torch.tensor(acts, dtype=torch.float32, device=dev).contiguous()
        env = pkg.Env(cfg, n, device=dev)
        env.reset()
        env.rollout(T, actions=a)
        torch.cuda.synchronize()
        reps = 5
        e0.record(stream)
        for _ in range(reps):
            env.rollout(T, actions=a)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[f"{name}_open_loop_rollout"] = {"value": n * T / (ms / 1e3), "unit": "env-steps/s", "us_per_step": ms * 1e3 / T,
                                            "workload": f"{n} envs x {T} steps, one l2f_rollout launch, recorded actions"}
        o = env.make_out(obs_core=True, reward=True, flags=True)
        s2 = torch.cuda.Stream(device=dev)
        s2.wait_stream(stream)
        with torch.cuda.stream(s2):  # warm-up outside capture
            for k in range(3):
                env.step(a[k], o)
        stream.wait_stream(s2)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for k in range(T):
                env.step(a[k], o)
        g.replay()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[f"{name}_step_graph"] = {"value": n * T / (ms / 1e3), "unit": "env-steps/s", "us_per_step": ms * 1e3 / T,
                                     "workload": f"{n} envs x {T} l2f_step launches in one CUDA graph"}
        del env, g
    return out


def c4_exact(pkg, inputs, torch, dev):
    """BASELINE configs[3] exactly: 2^20 envs x 1000 steps, fused MLP rollout (C4 features)."""
    stream = torch.cuda.current_stream()
    n, T = 1 << 20, 1000
    env = pkg.Env(inputs.config_c4(), n, device=dev)
    env.reset()
    pol = pkg.Policy(inputs.policy_weights(146, 64, seed=7, out_bias=inputs.hover_policy_bias()), device=dev)
    env.rollout(50, policy=pol)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record(stream)
    for _ in range(reps):
        env.rollout(T, policy=pol)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"value": n * T / (ms / 1e3), "unit": "env-steps/s", "ms": ms,
            "workload": "C4: 2^20 envs x 1000 steps fused actor-MLP rollout (146-64-64-4), noise, reward, termination, "
                        "auto-reset, disturbance"}


def secondary(pkg, inputs, torch, dev, pk, f_clk):
    """C3 single-step API (HBM roofline), C1/C2 (latency-bound), C4 exactly, and the open-loop
    dynamics mode."""
    out = small_configs(pkg, inputs, torch, dev)
    out["C4_mlp_rollout"] = c4_exact(pkg, inputs, torch, dev)
    torch.cuda.empty_cache()
    stream = torch.cuda.current_stream()
    # C3: 2^20 envs, DR, l2f_step, ring of 8 action buffers (16 MiB each; > L2 in total with state)
    n = 1 << 20
    cfg = inputs.config_c3()
    env = pkg.Env(cfg, n, device=dev)
    env.reset()
    acts = [torch.tensor(inputs.actions_near_hover(1, n, seed=100 + k)[0], dtype=torch.float32, device=dev)
            for k in range(8)]
    o = env.make_out(obs_core=True, reward=True, flags=True)
    for k in range(20):
        env.step(acts[k % 8], o)
    torch.cuda.synchronize()
    reps = 400
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(reps):
        env.step(acts[k % 8], o)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    rate = n / (ms / 1e3)
    gbs = STEP_BYTES_DR * n / (ms / 1e3) / 1e9
    out["C3_step_api"] = {"value": rate, "unit": "env-steps/s", "us_per_step": ms * 1e3,
                          "sim_seconds_per_wall_second": rate * DT,
                          "roofline": {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                                       "frac": gbs / pk["hbm_gbs"], "traffic": traffic("step"),
                                       "traffic_note": "DRAM read+write bytes of one launch (ncu --set full)",
                                       "bytes_per_env_step": STEP_BYTES_DR, "peak_source": pk["source"]}}
    # the same 400 steps replayed from a CUDA graph of 50 l2f_step launches (what a training loop
    # that captures its step does): no per-call launch gap, consecutive kernels back to back
    gs = torch.cuda.Stream(device=dev)
    gs.wait_stream(stream)
    with torch.cuda.stream(gs):
        env.step(acts[0], o)
    stream.wait_stream(gs)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for k in range(50):
            env.step(acts[k % 8], o)
    graph.replay()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps // 50):
        graph.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms_g = e0.elapsed_time(e1) / (reps // 50 * 50)
    gbs_g = STEP_BYTES_DR * n / (ms_g / 1e3) / 1e9
    out["C3_step_api"]["graph"] = {"value": n / (ms_g / 1e3), "unit": "env-steps/s", "us_per_step": ms_g * 1e3,
                                   "roofline_frac": gbs_g / pk["hbm_gbs"], "achieved_gbs": gbs_g,
                                   "workload": "the same steps replayed from a CUDA graph of 50 l2f_step launches"}
    del graph
    # e2e of the step API through host buffers (pinned): H2D actions, D2H obs/reward/flags
    ha = acts[0].cpu().pin_memory()
    hobs = torch.empty(18, n).pin_memory()
    hr = torch.empty(n).pin_memory()
    hf = torch.empty(n, dtype=torch.uint8).pin_memory()
    env.step_host(ha, hobs, hr, hf)
    t0 = time.perf_counter()
    for _ in range(20):
        env.step_host(ha, hobs, hr, hf)
    el = (time.perf_counter() - t0) / 20
    out["C3_step_api"]["e2e"] = {"value": n / el, "unit": "env-steps/s", "h2d_bytes_per_step": 16 * n,
                                 "d2h_bytes_per_step": 77 * n}
    # f2: reward recalculation over a device replay buffer of 2^24 transitions,
    # HBM-bound: s' 68 B + a' 16 B read, r 4 B written per transition
    m = 1 << 24
    g = torch.Generator(device=dev).manual_seed(5)
    sbuf = torch.rand(17, m, device=dev, generator=g) - 0.5
    abuf = torch.rand(4, m, device=dev, generator=g) * 2 - 1
    env.recompute_rewards(0, sbuf, abuf)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(10):
        env.recompute_rewards(250000, sbuf, abuf)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    gbs = 88 * m / (ms / 1e3) / 1e9
    out["recompute_rewards"] = {"value": m / (ms / 1e3), "unit": "transitions/s", "ms": ms,
                                "roofline": {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                                             "frac": gbs / pk["hbm_gbs"], "bytes_per_transition": 88}}
    del env, acts, o, sbuf, abuf
    torch.cuda.empty_cache()
    # open-loop dynamics-only mode (paper-comparable): 2^20 envs x 1000 steps, flags 0
    cfg = inputs.config_c1()
    n = 1 << 20
    env = pkg.Env(cfg, n, device=dev)
    env.reset()
    env.rollout(50)
    torch.cuda.synchronize()
    e0.record(stream)
    env.rollout(1000)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    rate = n * 1000 / (ms / 1e3)
    alu = SMS * 128 * f_clk / 1e12
    ops_dyn, ops_dyn_src = alu_ops("open_dyn")
    out["open_loop_dynamics"] = {"value": rate, "unit": "env-steps/s", "ms": ms,
                                 "workload": "2^20 envs x 1000 steps, Philox random actions, no noise/termination",
                                 "vs_paper_T2000": rate / 1.284e9,
                                 "roofline": {"bound": "alu", "achieved": ops_dyn * rate / 1e12,
                                              "peak": alu, "unit": "Tops/s",
                                              "frac": ops_dyn * rate / 1e12 / alu,
                                              "ops_per_env_step": ops_dyn, "ops_source": ops_dyn_src}}
    del env
    # the paper's own simulator benchmark shape: 8192 envs (64 blocks x 128 threads) x
    # 10^6 steps of forward dynamics, 100 Hz; here with Philox random actions, one rollout call
    n, T = 8192, 1_000_000
    env = pkg.Env(cfg, n, device=dev)
    env.reset()
    env.rollout(1000)
    torch.cuda.synchronize()
    e0.record(stream)
    env.rollout(T)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    rate = n * T / (ms / 1e3)
    out["paper_P165_shape"] = {"value": rate, "unit": "env-steps/s", "ms": ms,
                               "workload": "8192 envs x 1e6 steps, dynamics only (C1 flags), Philox random actions: "
                                           "the shape of the paper's T2000 measurement (P:165); latency-bound "
                                           "(256 warps on 592 schedulers)",
                               "vs_paper_T2000": rate / 1.284e9}
    del env
    # the full C5 env step without the actor MLP (Philox random actions), for the MLP's share
    n = 1 << 21
    env = pkg.Env(inputs.config_c5(), n, device=dev)
    env.reset()
    env.rollout(20)
    torch.cuda.synchronize()
    e0.record(stream)
    env.rollout(200)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out["open_loop_c5_features"] = {"value": n * 200 / (ms / 1e3), "unit": "env-steps/s", "ms": ms,
                                    "workload": "2^21 envs x 200 steps, C5 features, Philox random actions"}
    del env
    torch.cuda.empty_cache()
    # f3: batched Lissajous tracking (l2f_track), 2^20 envs sweeping the Table III cycle times
    n, steps = 1 << 20, 550
    cfg = inputs.config_c4()
    env = pkg.Env(cfg, n, device=dev)
    pol = pkg.Policy(inputs.policy_weights(146, 64, seed=7, out_bias=inputs.hover_policy_bias()), device=dev)
    ct = torch.tensor([15.0, 5.5, 3.5], device=dev).repeat(n // 3 + 1)[:n].contiguous()
    env.track(pol, ct, 20)
    torch.cuda.synchronize()
    e0.record(stream)
    r = env.track(pol, ct, steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ok = (r["steps_ok"] == steps)
    out["lissajous_tracking"] = {"value": n * steps / (ms / 1e3), "unit": "env-steps/s", "ms": ms,
                                 "workload": "2^20 envs x 550 steps (5.5 s), cycle times 15/5.5/3.5 s, random "
                                             "hover-biased C4 actor (untrained: RMSE values are not Table III's)",
                                 "success_fraction": float(ok.float().mean())}
    del env, pol, ct, r
    torch.cuda.empty_cache()
    # f4: batched TD3 update (l2f_td3_update), one agent per SM, B = 256, actor 146-64-64-4,
    # twin critics 32-64-64-1; a delayed (actor) step every second update (S:436 d = 2)
    A, B, I = SMS, 256, 146
    td3 = pkg.TD3(A, I, B, device=dev)
    g = torch.Generator(device=dev).manual_seed(3)
    td3.params.uniform_(-0.1, 0.1, generator=g)
    o = td3.offsets()
    td3.params[:, o["m_actor"]:].zero_()
    bt = {"o_a": torch.randn(A, B, I, device=dev, generator=g) * 0.5, "o_c": torch.randn(A, B, 28, device=dev, generator=g) * 0.5,
          "a": torch.rand(A, B, 4, device=dev, generator=g) * 2 - 1, "r": torch.randn(A, B, device=dev, generator=g),
          "o_a2": torch.randn(A, B, I, device=dev, generator=g) * 0.5, "o_c2": torch.randn(A, B, 28, device=dev, generator=g) * 0.5,
          "done": (torch.rand(A, B, device=dev, generator=g) < 0.1).float(), "eps": torch.randn(A, B, 4, device=dev, generator=g)}
    for k in range(4):
        td3.update(bt, update_actor=(k % 2 == 1))
    torch.cuda.synchronize()
    reps = 20
    e0.record(stream)
    for k in range(reps):
        td3.update(bt, update_actor=(k % 2 == 1))
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    # algorithmic FP32 work per sample (MAC = 2 flops): target actor + 2 target critics 26 112,
    # 2 x critic (forward 6 208 + deltas 4 160 + weight gradients 6 208) 33 152, and on the delayed
    # step actor forward 13 696 + Q1 forward/backward 12 416 + actor deltas 4 352 + gradients 13 696
    macs = B * (26112 + 33152 + 0.5 * (13696 + 12416 + 4352 + 13696))
    tf = A * 2 * macs / (ms / 1e3) / 1e12
    fp32_peak = SMS * 128 * 2 * f_clk / 1e12
    out["td3_update"] = {"value": A / (ms / 1e3), "unit": "agent-updates/s", "ms_per_call": ms,
                         "workload": f"{A} agents x batch {B}, actor {I}-64-64-4, twin critics 32-64-64-1, actor every 2nd",
                         "roofline": {"bound": "fp32", "achieved": tf, "peak": fp32_peak, "unit": "TFLOP/s",
                                      "frac": tf / fp32_peak, "peak_source": "148 SMs x 128 FP32 lanes x 2 x sampled clock"}}
    del td3, bt
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
