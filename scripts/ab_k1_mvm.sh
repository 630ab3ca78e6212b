#!/bin/bash
# same-box alternating A/B of one C3 matvec (prof_mvm.py, 8 reps each, last 6 reported) for two K1 builds
for rep in 1 2 3; do
  for v in "$@"; do
    echo -n "$v rep $rep: "
    CIQ_LIB=_ab/$v/libciq.so python scripts/prof_mvm.py --config C3 --reps 8 2>/dev/null | tail -6 | awk '{print $5}' | tr '\n' ' '
    echo
  done
done
