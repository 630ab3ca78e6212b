#!/bin/bash
# One GPU session: smoke, gpu tests, default bench, ncu launch list, ncu --set full of the top kernels.
# usage (on the box): bash scripts/gpu_round.sh [tag] [quick]
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi_$tag.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> $out/smoke_$tag.log
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu_$tag.log
timeout 600 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$tag.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $out/bench_ncu_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mvm_tc -s 3 -c 1 -f -o $out/k1_$tag \
  python scripts/prof_mvm.py --config C3 --reps 5 > $out/ncu_k1_$tag.log 2>&1
if [ "$2" != "quick" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lanczos_update_kernel -s 30 -c 1 -f -o $out/k4_$tag \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $out/ncu_k4_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mvm_dense -s 3 -c 1 -f -o $out/k2_$tag \
  python scripts/prof_mvm.py --config C2 --reps 5 > $out/ncu_k2_$tag.log 2>&1
fi
echo done
