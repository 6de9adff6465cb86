"""Per-CUDA-source-line stall-reason breakdown of an ncu report (--set full, source import).
usage: python scripts/ncu_stalls.py report.ncu-rep [reason] [top]
Prints the lines with the most samples of `reason` (default: all samples), with each line's
instructions and its share of every stall reason."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
reason = sys.argv[2] if len(sys.argv) > 2 else "Warp Stall Sampling (All Samples)"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, agg = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] in ("File Name", "File Path"):
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = {}
        for k, v in zip(hdr, r):
            try:
                d[k] = float(v)
            except ValueError:
                pass
        if d.get("Instructions Executed", 0) or d.get("Warp Stall Sampling (All Samples)", 0):
            agg.append((cur, r[0], r[1].strip()[:60], d))
reasons = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
tot = {k: sum(a[3].get(k, 0) for a in agg) for k in reasons + ["Warp Stall Sampling (All Samples)"]}
print("totals:", {k.replace("stall_", ""): round(100 * v / tot["Warp Stall Sampling (All Samples)"], 1)
                  for k, v in tot.items() if k in reasons and v})
key = reason if reason in tot else "stall_" + reason
for f, ln, src, d in sorted(agg, key=lambda a: -a[3].get(key, 0))[:top]:
    parts = " ".join(f"{k[6:]}={100 * d.get(k, 0) / tot['Warp Stall Sampling (All Samples)']:.2f}"
                     for k in reasons if d.get(k, 0) > 0.02 * d.get("Warp Stall Sampling (All Samples)", 1))
    print(f"{100 * d.get(key, 0) / max(tot[key], 1):5.1f}%  {f}:{ln} {src:60s} | {parts}")
