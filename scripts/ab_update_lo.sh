#!/bin/bash
# A/B of the Lanczos-only (stored-basis) streaming pass residency (CIQ_UPD_MINB_L) at C3.
for m in 3 4 5; do
  CIQ_LIB=_ab/updl_$m/libciq.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_updl_$m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_updl_$m.json')); print('MINB_L=$m', 'step ms', round(d['ms_per_step'],2), 'update us', round(1000*d['roofline_recurrence']['ms_per_launch'],1), 'mvm ms', round(d['roofline']['ms_per_launch'],4))"
done
