#!/bin/bash
# A/B (same box, alternating): K1 O slots alternating by unit (default) vs by tile within a unit
# (CIQ_TC2_ALT: 132-tile units = two 66-tile chains, half the units and half the partial products)
CIQ_LIB=_ab/k1_alt/libciq.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "tc or c3" 2>&1 | tail -1
for rep in 1 2; do
  for v in k1_def k1_alt; do
    CIQ_LIB=_ab/$v/libciq.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_${v}_$rep.json')); print('$v rep $rep', 'step ms', round(d['ms_per_step'],2), 'mvm ms', round(d['roofline']['ms_per_launch'],4), 'update us', round(1000*d['roofline_recurrence']['ms_per_launch'],1), 'splits', d['run']['mvm_splits'], 'mhz', d['clocks']['sm_mhz'])"
  done
done
