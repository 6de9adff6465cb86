"""Summarise the L2F_PHASE lines of a -DL2F_PHASE_TIMING run (cycles per tile-step per phase)."""
import sys

NAMES = ["obs", "bar1", "issue1+hook1", "wait1", "epi1", "bar2", "issue2+hook2", "wait2", "epi2", "bar3",
         "issue3+hook3", "wait3+tanh", "transition", "hist", "stats", "reset"]
rows = [list(map(int, l.split()[3:])) for l in open(sys.argv[1]) if l.startswith("L2F_PHASE")]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 200 * 28  # T x tile rounds per group (2^21 envs, 4 groups)
tot = [sum(r[k] for r in rows) / len(rows) for k in range(len(NAMES))]
s = sum(tot)
print(f"cycles per tile-step {s / steps:.0f}")
for n, v in zip(NAMES, tot):
    per_warp = [r[NAMES.index(n)] / steps for r in rows[:4]]
    print(f"{n:14s} {v / steps:7.0f} {v / s * 100:5.1f}%   warps0-3: " + " ".join(f"{x:6.0f}" for x in per_warp))
