"""Aggregate an ncu report's per-source-line instructions and stall samples by the device
function each line belongs to (function ranges parsed from the csrc sources).
usage: python scripts/ncu_regions.py report.ncu-rep [units]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2311_13081_b200", "csrc")


def function_ranges(path):
    """[(start_line, name)] for every function definition in a CUDA source file."""
    out = []
    pat = re.compile(r"^(?:template\s*<[^>]*>\s*)?(?:__global__|__device__|static|cudaError_t|int|bool)[\w\s:<>,\*&\(\)]*?\b(\w+)\s*\(")
    for no, line in enumerate(open(path), 1):
        m = pat.match(line)
        if m and not line.rstrip().endswith(";"):
            out.append((no, m.group(1)))
    return out


ranges = {f: function_ranges(os.path.join(CSRC, f)) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))}


def owner(fname, line):
    rs = ranges.get(fname)
    if not rs:
        return fname
    name = fname
    for start, n in rs:
        if start <= line:
            name = n
    return name


rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur, hdr = None, None
inst = collections.Counter()
samp = collections.Counter()
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            n = float(r[hdr.index("Instructions Executed")])
            s = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
            ln = int(r[0])
        except (ValueError, IndexError):
            continue
        key = owner(cur, ln)
        inst[key] += n
        samp[key] += s
ti, ts = sum(inst.values()), sum(samp.values())
print(f"{'function':28s} {'inst/unit':>10s} {'inst%':>6s} {'stall%':>7s}")
for k, _ in sorted(samp.items(), key=lambda kv: -kv[1])[:30]:
    print(f"{k:28s} {inst[k] / units:10.1f} {inst[k] / ti * 100:6.1f} {samp[k] / ts * 100:7.1f}")
