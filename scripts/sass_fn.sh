#!/bin/bash
# SASS of the kernels of libl2f.so whose mangled name contains $1 (e.g. rollout_mlp_kernelILb0ELi32ELb0ELj31)
cuobjdump -sass paper_2311_13081_b200/libl2f.so | awk -v pat="$1" '/Function : /{f = index($0, pat) > 0} f' | grep -v '^\s*/\* 0x'
