"""List the source lines of a kernel's local-memory spill instructions (STL/LDL).
usage: python scripts/spills.py <nvdisasm -gi output> <kernel name substring>"""
import collections
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lines = open(sys.argv[1]).read().split("\n")
cur, cnt, infn = None, collections.Counter(), False
for l in lines:
    if l.strip().startswith(".section") and ".text." in l:
        infn = sys.argv[2] in l
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.search(r"\b(STL|LDL)", l):
        cnt[(cur, "STL" if "STL" in l else "LDL")] += 1
for ((f, ln), kind), v in sorted(cnt.items(), key=lambda kv: -kv[1])[:40]:
    p = os.path.join(ROOT, "paper_2311_13081_b200", "csrc", f)
    txt = open(p).read().split("\n")[ln - 1].strip()[:80] if os.path.exists(p) else ""
    print(f"{v:3d} {kind} {f}:{ln}  {txt}")
