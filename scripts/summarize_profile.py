"""Write a markdown summary of a profiling pass (scripts/profile.sh) into profiles/<tag>/.

usage: python scripts/summarize_profile.py gpurun_out/prof_<tag> profiles/<tag>
Copies the launch list CSV and writes SUMMARY.md: per-kernel launch shares (serialised,
cold-cache ncu durations), key metrics of every --set full report, and the top CUDA source
lines by executed instructions."""
import collections
import csv
import io
import os
import shutil
import subprocess
import sys

src, dst = sys.argv[1], sys.argv[2]
os.makedirs(dst, exist_ok=True)
out = ["# Profile summary: " + os.path.basename(dst), ""]

# ---- launch list
lc = os.path.join(src, "launches.csv")
if os.path.exists(lc):
    shutil.copy(lc, os.path.join(dst, "launches.csv"))
    lines = [l for l in open(lc) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            agg[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    out += ["## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; serialised, cold cache)", "",
            "| kernel | launches | mean us | share of profiled time |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot * 100:.1f}% |")
    out.append("")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
]
traffic = {}
for rep in sorted(f for f in os.listdir(src) if f.endswith(".ncu-rep")):
    path = os.path.join(src, rep)
    shutil.copy(path, os.path.join(dst, rep))
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) < 3:
        continue
    h, u, v = rr[0], rr[1], rr[2]
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else rep
    try:
        rd = float(v[h.index("dram__bytes_read.sum")]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[
            u[h.index("dram__bytes_read.sum")]]
        wr = float(v[h.index("dram__bytes_write.sum")]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[
            u[h.index("dram__bytes_write.sum")]]
        traffic[rep.replace(".ncu-rep", "")] = {"kernel": name.split("(")[0], "dram_bytes": rd + wr,
                                                "dram_read": rd, "dram_write": wr}
    except (ValueError, KeyError):
        pass
    out += [f"## `{rep}`: {name.split('(')[0]}", "", "| metric | value |", "|---|---|"]
    for m in METRICS:
        if m in h:
            i = h.index(m)
            out.append(f"| {m} | {v[i]} {u[i]} |")
    out.append("")
    lines = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_lines.py"), path, "1", "25"],
                           capture_output=True, text=True).stdout
    out += ["Top CUDA source lines by executed warp-instructions:", "", "```", lines.rstrip(), "```", ""]
if os.path.exists(os.path.join(dst, "PHASES.md")):
    out += ["", "Per-phase cycle breakdowns from the debug builds: `PHASES.md` (same directory)."]
open(os.path.join(dst, "SUMMARY.md"), "w").write("\n".join(out) + "\n")
import json  # noqa: E402
json.dump(traffic, open(os.path.join(dst, "traffic.json"), "w"), indent=1)
# bench.py reports these per-launch DRAM bytes as roofline.traffic
json.dump({"source": os.path.join(dst, "traffic.json"), **traffic},
          open(os.path.join(os.path.dirname(dst.rstrip("/")), "latest_traffic.json"), "w"), indent=1)
print("\n".join(out))
