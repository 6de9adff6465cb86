"""Summarise an ncu report per CUDA source line: instructions executed and stall samples.
usage: python scripts/ncu_lines.py report.ncu-rep [units_for_normalisation] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = None
hdr = None
agg = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            inst = float(r[hdr.index("Instructions Executed")])
            samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        agg.append((inst, samp, cur, r[0], r[1][:70]))
tot_i = sum(a[0] for a in agg)
tot_s = sum(a[1] for a in agg)
print(f"total warp-instructions {tot_i:.4g}  per unit {tot_i / units:.1f}")
for inst, samp, f, ln, src in sorted(agg, reverse=True)[:top]:
    print(f"{inst / units:8.1f} {inst / tot_i * 100:5.1f}% stall {samp / tot_s * 100:5.1f}%  {f}:{ln}  {src}")
