#!/bin/bash
# A/B (same box, alternating): dense path with / without the level-2 relaxation (K_hi planes only
# once relres <= 0.01), C2; plus the GPU tests on the new build
CIQ_LIB=_ab/drelax/libciq.so timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do for v in dbase drelax; do
  CIQ_LIB=_ab/$v/libciq.so timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v rep $rep step ms', round(d['ms_per_step'],3), 'value', round(d['value'],1), 'J', d['run']['J'], 'r2', d['run'].get('relaxed2_from_step'))"
done; done
