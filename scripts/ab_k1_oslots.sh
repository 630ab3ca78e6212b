#!/bin/bash
# A/B (same box, alternating): K1 with 3 S/K TMEM buffers + one O slot (default) vs 2 S/K buffers +
# two O slots (the next unit's first KV never waits for the read-out), C3.
CIQ_LIB=_ab/k1_nb2o2/libciq.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tc" 2>&1 | tail -1
for rep in 1 2; do
  for v in k1_nb3o1 k1_nb2o2; do
    CIQ_LIB=_ab/$v/libciq.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_${v}_$rep.json')); print('$v rep $rep', 'step ms', round(d['ms_per_step'],2), 'mvm ms', round(d['roofline']['ms_per_launch'],4), 'mhz', d['clocks']['sm_mhz'])"
  done
done
