#!/bin/bash
# A/B of K1 library variants on one box: bash scripts/ab_variants.sh "base trunc hint both" [config]
vars=${1:-"base trunc hint both"}; cfg=${2:-C3}
for round in 1 2 3; do
  for v in $vars; do
    echo -n "$v round $round: "
    CIQ_LIB=_ab/$v/libciq.so timeout 120 python scripts/prof_mvm.py --config $cfg --reps 8 | tail -4 | awk '{s+=$(NF-3)} END {printf "%.4f ms (mean of last 4)\n", s/4}'
  done
done
