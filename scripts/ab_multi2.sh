# A/B of several library variants on one box: bash scripts/ab_multi2.sh "<cfg> <impl> <t>" V1 V2 ...
# (variants in _ab/<V>/libciq.so; interleaved rounds, mean of the last 4 of 6 reps)
spec=$1; shift
set -- $spec "$@"; cfg=$1; impl=$2; t=$3; shift 3
for round in 1 2 3; do
  for v in "$@"; do
    echo -n "$cfg $impl t=$t $v round $round: "
    CIQ_LIB=_ab/$v/libciq.so timeout 120 python scripts/prof_mvm.py --config $cfg --impl $impl --t $t --reps 6 | tail -4 | awk '{s+=$(NF-3)} END {printf "%.4f ms\n", s/4}'
  done
done
