#!/bin/bash
# Step-level A/B between library builds: bash scripts/ab_bench.sh "base qb2" [config]
vars=${1:-"base"}; cfg=${2:-C3}
for round in 1 2; do
  for v in $vars; do
    CIQ_LIB=_ab/$v/libciq.so timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d.get('roofline_recurrence',{})
print('$v round $round: %.2f ms/step  %.1f RHS/s  K1 %.3f ms  update %.1f us' % (d['ms_per_step'], d['value'], d['roofline']['ms_per_launch'], 1000*r.get('ms_per_launch',0)))"
  done
done
