#!/bin/bash
# Evidence run for profiles/ (one B200): bench lines for every config and the reference arm,
# the cfg5 launch list, and one `ncu --set full` capture of each hot kernel.
#   tools/round_evidence.sh <tag>      (writes gpurun_out/<tag>_*)
set -u
T=${1:-r2b}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${T}_smi.txt 2>&1
for c in 5 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $O/${T}_bench_cfg$c.log 2>&1; echo "bench cfg$c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${T}_bench_reference_cfg5.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv --log-file $O/${T}_launches_cfg5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-per-metric > $O/${T}_ncu_launch.log 2>&1; echo "launch rc=$?"
for k in k_pairs_lag1 k_pairs_tc k_spectra_dmma; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $O/${T}_$k \
    python tools/prof_run.py --config 5 --reps 2 > $O/${T}_ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
