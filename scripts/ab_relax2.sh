#!/bin/bash
# A/B (same box, alternating): relaxed schedule level 1 only (long chains from relres 0.1) vs level 2
# (also k_hi-only MVMs from relres 0.01); C3 golden error and throughput
for v in lvl1 lvl2; do
  echo "$v: $(CIQ_LIB=_ab/$v/libciq.so timeout 300 python scripts/diag_chain_nsplit.py 2>&1 | grep nsplit | sed 's/.* invsqrt=/invsqrt=/' | cut -c1-300)"
done
for rep in 1 2; do for v in lvl1 lvl2; do
  CIQ_LIB=_ab/$v/libciq.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v rep $rep step ms', round(d['ms_per_step'],2), 'value', round(d['value'],1), 'run', d['run'].get('relaxed_from_step'), 'mhz', d['clocks']['sm_mhz'])"
done; done
