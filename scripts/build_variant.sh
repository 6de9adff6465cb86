#!/bin/bash
# Build libl2f.so with extra nvcc defines into build/ab/libl2f_<tag>.so (A/B experiments),
# then restore the default build.  Usage: scripts/build_variant.sh <tag> "<defines>"
set -e
tag=$1; defs=${2:-}
L2F_NVCC_DEFS="$defs" python -c "from paper_2311_13081_b200 import _build; _build.build(force=True)" 2>&1 | grep -E "error|rollout_mlp_kernelILb0ELi32|spill" | grep -B1 -A0 spill | head -4 || true
mkdir -p build/ab
cp paper_2311_13081_b200/libl2f.so build/ab/libl2f_$tag.so
