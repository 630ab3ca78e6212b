#!/bin/bash
# A/B (same box, alternating): alpha in the full-tile MVM's tail vs the separate alpha pass, C3 and C2.
for rep in 1 2; do
  for v in afuse anofuse; do
    for c in C3 C2; do
      CIQ_LIB=_ab/$v/libciq.so timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${v}_${c}_$rep.json 2>/dev/null
      python -c "import json; d=json.load(open('gpurun_out/ab_${v}_${c}_$rep.json')); print('$v $c rep $rep', 'step ms', round(d['ms_per_step'],2), 'mvm ms', round(d['roofline']['ms_per_launch'],4), 'launches', d['gpu_launches'], 'mhz', d['clocks']['sm_mhz'])"
    done
  done
done
