#!/bin/bash
# Session 14: the final library (warp pair for n = 52..64; 2 terms per exchange from n = 60) --
# warp-pair parity tests, the whole GPU suite with the tolerance report, smoke, the three-way A/B
# (wsplit_bench), library rates at n = 52..64 on 888 custom units, ncu --set full of
# wsplit_kernel<64> (the 2-terms-per-exchange body).
set -u
O=gpurun_out/r02s14; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_wsplit.py -q > $O/pytest_wsplit.log 2>&1; echo "pytest_wsplit rc=$?" >> $O/status.txt
PERMB200_TOL_REPORT=$O/tol_report.json timeout 1500 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 600 tools/microbench/wsplit_bench 2 > $O/wsplit_bench.log 2>&1; echo "wsplit_bench rc=$?" >> $O/status.txt
for n in 52 54 56 58 59 60 61 62 63 64; do
  for alg in glynn ryser; do
    [ "$n$alg" = "64ryser" ] && continue
    timeout 300 python tools/profile_sweep.py --custom 11,4,6 --units 888 --reps 3 --n $n --alg $alg >> $O/large_n.log 2>&1
  done
done
echo "large_n done" >> $O/status.txt
P64="python tools/profile_sweep.py --n 64 --custom 11,4,6 --units 296 --reps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wsplit_kernel -c 1 -o $O/wsplit_n64 $P64 > $O/ncu64.log 2>&1; echo "ncu64 rc=$?" >> $O/status.txt
echo "pre14 done $(date)" >> $O/status.txt
