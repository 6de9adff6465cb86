"""After scripts/prof_round.sh <tag>: summarise the captures into profiles/<tag>/ (SUMMARY.md,
launch list, DRAM traffic) and write the mechanical ALU work counts (scripts/alu_ops.py) into
profiles/<tag>/alu_ops_*.json and profiles/alu_ops.json (read by bench.py).
usage: python scripts/finish_profiles.py <tag>"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src, dst = os.path.join(ROOT, "gpurun_out", "prof_" + tag), os.path.join(ROOT, "profiles", tag)
subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "summarize_profile.py"), src, dst], check=True,
               capture_output=True)
# env-steps in each capture (the workloads of scripts/prof_round.sh)
caps = {"mlp": ("mlp.ncu-rep", (1 << 21) * 1000), "open_dyn": ("open_dyn.ncu-rep", (1 << 20) * 1000),
        "open_c5": ("open_c5.ncu-rep", (1 << 21) * 200), "step": ("step.ncu-rep", 1 << 20)}
out = {}
lines = ["", "## Mechanical ALU work counts (scripts/alu_ops.py)", "",
         "| kernel | method ops / env-step | all (per-PC counts) | all (smsp__inst_executed) | UTCHMMA | LDTM | STTM | MUFU |",
         "|---|---|---|---|---|---|---|---|"]
for k, (rep, units) in caps.items():
    path = os.path.join(src, rep)
    if not os.path.exists(path):
        continue
    js = os.path.join(dst, f"alu_ops_{k}.json")
    subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "alu_ops.py"), path, str(units), js], check=True,
                   capture_output=True)
    d = json.load(open(js))
    d["report"] = os.path.join("profiles", tag, rep)
    json.dump(d, open(js, "w"), indent=1)
    out[k] = {"method_ops_per_env_step": d["method_ops_per_env_step"], "total_per_env_step": d["total_per_env_step"],
              "smsp_inst_executed_per_env_step": d.get("smsp_inst_executed_per_env_step"),
              "source": f"profiles/{tag}/alu_ops_{k}.json (scripts/alu_ops.py over the {rep} capture)"}
    h = d["sass_histogram_per_env_step"]
    sm = d.get("smsp_inst_executed_per_env_step")
    lines.append(f"| {k} | {d['method_ops_per_env_step']:.0f} | {d['total_per_env_step']:.0f} | "
                 f"{sm:.0f} | {h['UTCHMMA']:.2f} | "
                 f"{h['LDTM']:.2f} | {h['STTM']:.2f} | {h['MUFU']:.1f} |")
lines += ["", "Counts are per env-step (warp-instructions per 32 env-steps); the SASS columns are executed "
              "instructions of those opcodes per env-step (tcgen05.mma = UTCHMMA, tcgen05.ld/st = LDTM/STTM).  "
              "The per-PC counts come from an instrumented replay in which barrier / mbarrier wait loops spin "
              "more often than in the plain run (smsp__inst_executed); the method count has no wait loops."]
json.dump(out, open(os.path.join(ROOT, "profiles", "alu_ops.json"), "w"), indent=1)
with open(os.path.join(dst, "SUMMARY.md"), "a") as f:
    f.write("\n".join(lines) + "\n")
print(json.dumps(out, indent=1))
