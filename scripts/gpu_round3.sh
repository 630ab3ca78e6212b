#!/bin/bash
# Round-2 final GPU session: smoke, gpu tests, benches (C3 default + C2/C4/C5/T1/G1 + reference),
# ncu launch list of the default bench, ncu --set full of K1 (C3), the fp64 DMMA M MVM (C4) and the
# stored-basis update kernel (C3).   usage (on the box): bash scripts/gpu_round3.sh <tag>
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/smi_$tag.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> $out/smoke_$tag.log
timeout 2000 python -m pytest tests -m gpu -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu_$tag.log
timeout 900 python bench.py > $out/bench_${tag}_c3.json 2> $out/bench_${tag}_c3.err
for c in C2 C4 C5 T1 G1; do
  timeout 900 python bench.py --config $c > $out/bench_${tag}_$(echo $c | tr A-Z a-z).json 2> $out/bench_${tag}_$c.err
done
timeout 900 python bench.py --impl reference > $out/bench_${tag}_ref.json 2> $out/bench_${tag}_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$tag.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $out/bench_ncu_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mvm_tc2 -s 3 -c 1 -f -o $out/k1_$tag \
  python scripts/prof_mvm.py --config C3 --reps 5 > $out/ncu_k1_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mvm64 -s 12 -c 1 -f -o $out/k64_$tag \
  python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline > $out/ncu_k64_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lanczos_update_kernel -s 30 -c 1 -f -o $out/k4s_$tag \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --recurrence stored > $out/ncu_k4s_$tag.log 2>&1
echo done
