#!/bin/bash
# Session 7 pre-script: M1 anatomy (phase timers, double-buffered vs in-place walk), the GPU
# parity suite on the rebuilt library (small n back to one lane per chunk + double buffer),
# M1 latency through the library.
set -u
O=gpurun_out/r02s7; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
for v in db1t db0t db1 db0 db1t db0t; do echo "== $v" >> $O/m1_phases.log; timeout 120 tools/microbench/m1_phases_$v >> $O/m1_phases.log 2>&1; done
echo "m1 phases done" > $O/status.txt
for v in c0mb4 db2 db3 c0mb4 db2 db3; do echo "v $v" >> $O/batched_variants.log; timeout 120 tools/microbench/batched_bench_$v 4096 >> $O/batched_variants.log 2>&1; done
PERMB200_TOL_REPORT=$O/tol_report.json timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python tools/latency_probe.py > $O/latency.log 2>&1; echo "latency rc=$?" >> $O/status.txt
timeout 300 python tools/r02/m1_plans.py > $O/m1_plans_glynn.log 2>&1; echo "m1g rc=$?" >> $O/status.txt
timeout 300 python tools/r02/m1_plans.py --alg ryser > $O/m1_plans_ryser.log 2>&1; echo "m1r rc=$?" >> $O/status.txt
echo "pre7 done $(date)" >> $O/status.txt
