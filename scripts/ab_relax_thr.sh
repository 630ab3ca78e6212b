#!/bin/bash
# C3: relaxed-schedule threshold vs golden error and throughput (experiments build, CIQ_RELAX_THR)
for thr in 0.1 0.25 0.5; do
  echo "thr $thr: $(CIQ_LIB=_ab/exp/libciq.so CIQ_RELAX_THR=$thr timeout 300 python scripts/diag_chain_nsplit.py 2>&1 | grep nsplit | sed 's/.*sqrt=/sqrt=/' | cut -c1-300)"
done
for rep in 1 2; do for thr in 0.1 0.25 0.5; do
  CIQ_LIB=_ab/exp/libciq.so CIQ_RELAX_THR=$thr timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_thr_$thr.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_thr_$thr.json')); print('thr $thr rep $rep step ms', round(d['ms_per_step'],2), 'relaxed_from', d['run']['relaxed_from_step'], 'mhz', d['clocks']['sm_mhz'])"
done; done
