#!/bin/bash
# Session 8 pre-script: A/B of the loop-carried step-0 row (PERMB200_ROW_AHEAD, sweep_bench
# n = 32/40/50), then the GPU parity suite and the bench line on the rebuilt library.
set -u
O=gpurun_out/r02s8; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
for v in ra1 ra0 c5a1 c5a0 ra1 ra0 c5a1 c5a0; do echo "== $v" >> $O/sweep_ab.log; timeout 300 tools/microbench/sweep_bench_$v 8 >> $O/sweep_ab.log 2>&1; done
echo "ab done" > $O/status.txt
PERMB200_TOL_REPORT=$O/tol_report.json timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?" >> $O/status.txt
timeout 300 python tools/latency_probe.py > $O/latency.log 2>&1; echo "latency rc=$?" >> $O/status.txt
echo "pre8 done $(date)" >> $O/status.txt
