#!/bin/bash
# Round-2 evidence pass (session 5, after the container was re-created): full GPU parity suite
# with the tolerance report, the bench line, M1 latency, batched >= 1e5 run, Table AV, 2-rank
# gloo bench, bounds-checked build + determinism stress.  Then the caller runs a Ryser segment
# session of the remaining budget.
set -u
O=gpurun_out/r02s5; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
PERMB200_TOL_REPORT=$O/tol_report.json timeout 1500 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" > $O/status.txt
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?" >> $O/status.txt
timeout 300 python tools/latency_probe.py > $O/latency.log 2>&1; echo "latency rc=$?" >> $O/status.txt
timeout 300 python tools/r02/m1_plans.py > $O/m1_plans_glynn.log 2>&1; echo "m1g rc=$?" >> $O/status.txt
timeout 600 python tools/r02/batched_run.py --out $O/batched.json > $O/batched.log 2>&1; echo "batched rc=$?" >> $O/status.txt
timeout 900 python tools/r02/table_av.py --out $O/r02_precision > $O/table_av.log 2>&1; echo "tableav rc=$?" >> $O/status.txt
PERMB200_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 2 --warmup 3 > $O/bench_gloo2.json 2> $O/bench_gloo2.err; echo "bench2 rc=$?" >> $O/status.txt
bash tools/r02/checked.sh; cp -r gpurun_out/r02_checked $O/ 2>/dev/null
echo "pre5 done $(date)" >> $O/status.txt
