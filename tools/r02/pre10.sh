#!/bin/bash
# Session 10 pre-script (re-created container): GPU parity suite on the current tree (small-n
# build + shuffle-tree changes), smoke, the default bench line; then the ladder continues.
set -u
O=gpurun_out/r02s10; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
PERMB200_TOL_REPORT=$O/tol_report.json timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
timeout 300 python tools/latency_probe.py > $O/latency.log 2>&1; echo "latency rc=$?" >> $O/status.txt
echo "pre10 done $(date)" >> $O/status.txt
