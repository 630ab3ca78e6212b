# A/B the matrix-free MVM across library builds _ab/<name>/libciq.so on one box, interleaved rounds.
# usage: bash scripts/ab_multi.sh <config> <name> [<name> ...]
cfg=$1; shift
for round in 1 2 3; do
  for v in "$@"; do
    echo -n "$v round $round: "
    CIQ_LIB=_ab/$v/libciq.so timeout 120 python scripts/prof_mvm.py --config $cfg --reps 8 | tail -4 | awk '{s+=$(NF-3)} END {printf "%.4f ms (mean of last 4)\n", s/4}'
  done
done
