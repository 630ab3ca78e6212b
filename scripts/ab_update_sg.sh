#!/bin/bash
# A/B of the streaming-update kernel's launch bounds / grouped partial-product loads at C3 (stored
# basis, 12 column splits): per-launch update time from bench.py's profiled call.
# build (here): for v in "3 1" "2 1" "2 4" "3 2"; do set -- $v; python scripts/build_variant.py upd_m$1_g$2 -DCIQ_UPD_MINB=$1 -DCIQ_UPD_SG=$2; done
for v in upd_m3_g1 upd_m2_g1 upd_m2_g4 upd_m3_g2; do
  CIQ_LIB=_ab/$v/libciq.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', 'step ms', round(d['ms_per_step'],2), 'update us', round(1000*d['roofline_recurrence']['ms_per_launch'],1), 'mvm ms', round(d['roofline']['ms_per_launch'],4))"
done
