#!/bin/bash
# actor-MLP kernel family A/B (scripts/time_mlp_family.py) of build/ab/libl2f_<tag>.so, alternating twice
for rep in 1 2; do
for t in "$@"; do
  cp build/ab/libl2f_$t.so paper_2311_13081_b200/libl2f.so
  python scripts/time_mlp_family.py | sed "s/^/$t /"
done
done
