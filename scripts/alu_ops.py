"""Mechanical per-env-step operation count of a kernel from its ncu --set full capture (the
ALU roofline's algorithmic work).

usage: python scripts/alu_ops.py report.ncu-rep <env_steps_in_capture> <out.json>

Every executed SASS instruction of the capture is attributed (ncu source page, cuda + sass
view) to the CUDA source line it came from and that line to the device function enclosing it
(function ranges parsed from paper_2311_13081_b200/csrc).  An instruction counts as the
method's arithmetic when
  * its function is one of METHOD_FUNCTIONS (the steps of SURVEY 8(a): noise RNG and Box-Muller,
    observation, the fp16 quantisation and activations of the actor MLP, dynamics / RK4,
    reward, termination, reset sampling, episode statistics) or it is inlined from a CUDA math
    header (packed FP32, fp16 conversion), and
  * its opcode is an arithmetic, conversion, comparison or special-function opcode (not a move,
    constant load, branch, barrier, shuffle, memory access or MMA-issue opcode);
  * or it is an fp16 conversion (F2FP: the method's quantisation points, Q21).
Everything else -- MMA issue and hand-offs, TMEM / shared / global data movement, address
arithmetic, reset bookkeeping, control flow, moves -- is overhead.  The count is in
warp-instructions per 32 env-steps = lane-instructions per env-step, i.e. issue slots, against
an issue peak of one instruction per lane per cycle (148 SMs x 128 lanes x clock).  Packed
FFMA2 / FADD2 / FMUL2 count once (one issue slot).  Also writes the executed-count histogram
of the tensor-core / TMEM / TMA opcodes (UTCHMMA, UTCBAR, LDTM, STTM, UTMALDG, ...)."""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
CSRC = os.path.join(ROOT, "paper_2311_13081_b200", "csrc")

METHOD_FUNCTIONS = {
    # RNG (Q20) and Box-Muller
    "philox", "philox_rk", "draw", "unif", "ln_unit", "box_muller", "box_muller2", "obs_noise_blocks",
    "action_noise", "random_action", "uab",
    # observation, actor MLP activations / fp16 quantisation (Q21)
    "observe_core_z", "observe_core", "observe_critic", "add_obs_noise", "tanh_fast", "relu_pack", "pack_h2",
    # dynamics, RK4, reward, termination
    "make_phys", "deriv", "pair_fma", "rk4_step", "state_finite", "stepped_state_finite", "transition",
    "reward_of", "stage_of",
    # reset sampling, episode statistics
    "reset_block", "reset_values", "reset_values_tab", "reset_finish", "reset_env",
    "statpk_episode", "stat_episode",
}
MATH_HEADERS = ("sm_100_rt.hpp", "cuda_fp16.hpp", "math_functions.hpp", "device_functions.hpp",
                "sm_20_intrinsics.hpp_math")  # (sm_20 / sm_30 intrinsics are cvta / shuffles: overhead)
NON_ARITH = re.compile(r"^(MOV|IMAD\.MOV|UMOV|MOV32I|CS2R|S2R|S2UR|LDC|LDCU|ULDC|BRA|BSSY|BSYNC|BREAK|WARPSYNC|NOP|"
                       r"EXIT|RET|CALL|YIELD|BAR|SYNCS|R2UR|SHFL|VOTE|VOTEU|ELECT|MEMBAR|FENCE|ERRBAR|"
                       r"LD|ST|LDS|STS|LDG|STG|LDL|STL|LDTM|STTM|UTC|UTMA|REDUX|CCTL|PLOP3|UPLOP3|"
                       r"U[A-Z0-9]+)")
# fp16 conversions are always the method's quantisation (Q21: observation, history entries, the
# ReLU + round of the hidden layers); inline-asm ones carry their caller's line, so by opcode.
ALWAYS_METHOD = ("F2FP",)
SASS_CLASSES = ("UTCHMMA", "UTCBAR", "UTCATOMSWS", "LDTM", "STTM", "UTMALDG", "UTMASTG", "SYNCS", "BAR", "LDS", "STS",
                "LDG", "STG", "MUFU", "FFMA2", "FADD2", "FMUL2", "F2FP", "IMAD.WIDE")


def function_ranges(path):
    out = []
    pat = re.compile(r"^(?:template\s*<[^>]*>\s*)?(?:__global__|__device__|static|cudaError_t|int|bool)"
                     r"[\w\s:<>,\*&\(\)]*?\b(\w+)\s*\(")
    for no, line in enumerate(open(path), 1):
        m = pat.match(line)
        if m and not line.rstrip().endswith(";"):
            out.append((no, m.group(1)))
    return out


RANGES = {f: function_ranges(os.path.join(CSRC, f)) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))}


def owner(fname, line):
    rs = RANGES.get(fname)
    if not rs:
        return fname
    name = fname
    for start, n in rs:
        if start <= line:
            name = n
    return name


def opcode(sass):
    t = sass.strip().split()
    if not t:
        return ""
    if t[0].startswith("@"):
        t = t[1:]
    return t[0] if t else ""


def main():
    rep, units, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    # the cuda + sass view lists an inlined instruction under every source line of its inline call
    # stack: collect, per SASS address, the enclosing functions of all those lines
    cur, hdr, line_owner = None, None, None
    owners, info = collections.defaultdict(set), {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or not r:
            continue
        if r[0].isdigit():  # a CUDA source line; its SASS rows follow
            line_owner = (cur, owner(cur, int(r[0])))
            continue
        if len(r) < 8 or not r[2].startswith("0x"):
            continue
        try:
            n = float(r[hdr.index("Instructions Executed", 2)])
        except (ValueError, IndexError):
            continue
        owners[r[2]].add(line_owner)
        info[r[2]] = (n, opcode(r[3]))
    method, overhead = collections.Counter(), collections.Counter()
    by_func = collections.Counter()
    hist = collections.Counter()
    total = 0.0
    for addr, (n, op) in info.items():
        if n == 0:
            continue
        total += n
        for c in SASS_CLASSES:
            if op == c or op.startswith(c + "."):
                hist[c] += n
        fns = [fn for (f, fn) in owners[addr] if fn in METHOD_FUNCTIONS]
        hdrs = [f for (f, fn) in owners[addr] if (f or "").endswith(MATH_HEADERS)]
        if ((fns or hdrs) and not NON_ARITH.match(op)) or op.startswith(ALWAYS_METHOD):
            method[op.split(".")[0]] += n
            by_func[fns[0] if fns else (hdrs[0] if hdrs else "fp16 conversion")] += n
        else:
            overhead[op.split(".")[0]] += n
    warp_steps = units / 32.0
    units = warp_steps  # per-env-step lane-instructions = warp-instructions per warp-step
    m, o = sum(method.values()), sum(overhead.values())
    res = {"report": os.path.relpath(rep, ROOT), "env_steps": units * 32.0,
           "method_ops_per_env_step": m / units,
           "overhead_per_env_step": o / units, "total_per_env_step": total / units,
           "note": "warp-instructions per 32 env-steps (= lane-instructions per env-step); method = arithmetic "
                   "opcodes in the method's device functions (scripts/alu_ops.py docstring)",
           "method_by_opcode": {k: v / units for k, v in method.most_common()},
           "method_by_function": {k: v / units for k, v in by_func.most_common()},
           "overhead_by_opcode": {k: v / units for k, v in overhead.most_common(25)},
           "sass_histogram_per_env_step": {k: hist[k] / units for k in SASS_CLASSES},
           "sass_histogram_executed": {k: hist[k] for k in SASS_CLASSES}}
    # the whole-kernel executed-instruction metric of the same capture (the per-PC counts above come
    # from an instrumented replay, where mbarrier / barrier wait loops spin more often)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    try:
        res["smsp_inst_executed_per_env_step"] = float(rr[2][rr[0].index("smsp__inst_executed.sum")]) / units
    except (ValueError, IndexError):
        pass
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: res.get(k) for k in ("method_ops_per_env_step", "overhead_per_env_step", "total_per_env_step",
                                              "smsp_inst_executed_per_env_step")}))


if __name__ == "__main__":
    main()
