#!/bin/bash
# Session 9 pre-script: M1 anatomy after the small-n build + shuffle-tree changes (b1 vs b0 =
# old build), GPU parity suite, M1 latency through the library, FP64 issue vs warps/ILP probe.
set -u
O=gpurun_out/r02s9; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
for v in b1 b0 b1 b0; do echo "== $v" >> $O/m1_phases.log; timeout 120 tools/microbench/m1_phases_$v >> $O/m1_phases.log 2>&1; done
timeout 120 tools/microbench/fp64_warps > $O/fp64_warps.log 2>&1
echo "micro done" > $O/status.txt
PERMB200_TOL_REPORT=$O/tol_report.json timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python tools/latency_probe.py > $O/latency.log 2>&1; echo "latency rc=$?" >> $O/status.txt
timeout 300 python tools/r02/m1_plans.py > $O/m1_plans_glynn.log 2>&1; echo "m1g rc=$?" >> $O/status.txt
echo "pre9 done $(date)" >> $O/status.txt
