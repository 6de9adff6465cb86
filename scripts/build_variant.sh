#!/bin/bash
# Build libl2f.so with extra nvcc defines into build/ab/libl2f_<tag>.so (A/B experiments),
# then rebuild the default in-tree library.  Usage: scripts/build_variant.sh <tag> "<defines>"
set -e
tag=$1; defs=${2:-}
mkdir -p build/ab
L2F_NVCC_DEFS="$defs" python -c "from paper_2311_13081_b200 import _build; _build.build(force=True, verbose=True)" > build/ab/build_$tag.log 2>&1
cp paper_2311_13081_b200/libl2f.so build/ab/libl2f_$tag.so
python -c "from paper_2311_13081_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
grep -A2 "rollout_mlp_kernelILb0ELi32" build/ab/build_$tag.log | grep -E "spill|registers" | head -2 || true
