#!/bin/bash
# A/B of library variants: for each build/ab/libl2f_<tag>.so given, run the quick bench.
for tag in "$@"; do
  cp build/ab/libl2f_$tag.so paper_2311_13081_b200/libl2f.so
  echo "== $tag"; bash scripts/quick.sh
done
