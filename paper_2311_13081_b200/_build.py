"""Build libl2f.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libl2f.so")
SOURCES = ["l2f_abi.cu", "l2f_kernels.cu", "l2f_mlp.cu", "l2f_td3.cu"]
HEADERS = ["l2f_device.cuh", "l2f_internal.h", "l2f_tcgen05.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-ftz=true", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]
# Per-source extra flags (overridable per file with L2F_NVCC_<NAME>, e.g. L2F_NVCC_L2F_TD3): ptxas
# register-usage levels chosen by measurement (scripts/ab/all_ab.sh).
PER_SOURCE = {"l2f_mlp.cu": "-Xptxas --register-usage-level=8",  # rollout +0.5-1 %
              "l2f_td3.cu": "-Xptxas --register-usage-level=3"}  # TD3 +1 %


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "l2f.h"),
                                                                 os.path.abspath(__file__)]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    extra = os.environ.get("L2F_NVCC_DEFS", "").split()  # experiments only, e.g. -DL2F_MLP_TILES=4
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        per = os.environ.get("L2F_NVCC_" + src.replace(".cu", "").upper(), PER_SOURCE.get(src, "")).split()
        cmd = [NVCC, *ARCH, *FLAGS, *per, *extra, "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src),
               "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed for {src}")
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl",
           "-lpthread"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
