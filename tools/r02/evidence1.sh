#!/bin/bash
# Round-2 first GPU pass: parity suite, then refreshed ncu --set full captures of the kernels
# that carry the metric (each command first run clean without ncu).
set -u
OUT=gpurun_out/r02a
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" > $OUT/status.txt
P50G="python tools/profile_sweep.py --workload M5 --custom 11,4,7 --units 296 --reps 1"
P50R="python tools/profile_sweep.py --workload M5 --alg ryser --custom 11,4,7 --units 296 --reps 1"
PB="python tools/profile_sweep.py --workload M2 --batched --reps 1"
PDD="python tools/profile_sweep.py --workload M3 --alg glynn_dd --fraction 16 --reps 1"
for c in "$P50G" "$P50R" "$PB" "$PDD"; do $c >> $OUT/plain_runs.log 2>&1; echo "plain rc=$? $c" >> $OUT/status.txt; done
NCU="ncu --set full --clock-control none --import-source on -c 1"
$NCU -k regex:sweep_kernel -o $OUT/sweep_n50_glynn $P50G > $OUT/ncu1.log 2>&1; echo "ncu50g rc=$?" >> $OUT/status.txt
$NCU -k regex:sweep_kernel -o $OUT/sweep_n50_ryser $P50R > $OUT/ncu2.log 2>&1; echo "ncu50r rc=$?" >> $OUT/status.txt
$NCU -k regex:batched_kernel -o $OUT/batched_m2 $PB > $OUT/ncu3.log 2>&1; echo "ncub rc=$?" >> $OUT/status.txt
$NCU -k regex:sweep_dd -o $OUT/dd_n32 $PDD > $OUT/ncu4.log 2>&1; echo "ncudd rc=$?" >> $OUT/status.txt
