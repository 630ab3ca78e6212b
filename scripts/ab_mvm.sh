# A/B the matrix-free MVM between two library builds on the same box: _ab/A/libciq.so vs _ab/B/libciq.so
# usage: bash scripts/ab_mvm.sh [config] [t]
cfg=${1:-C3}; t=${2:-0}
for round in 1 2 3; do
  for v in A B; do
    echo -n "$v round $round: "
    CIQ_LIB=_ab/$v/libciq.so timeout 120 python scripts/prof_mvm.py --config $cfg --t $t --reps 8 | tail -4 | awk '{s+=$(NF-3)} END {printf "%.4f ms (mean of last 4)\n", s/4}'
  done
done
