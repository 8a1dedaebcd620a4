#!/bin/bash
# Session 12 pre-script: the warp-pair split after its first GPU run (n = 52..60 on the warp pair,
# n = 61..64 back on the 2-lane split; test fix) -- its parity tests, the whole GPU suite with the
# tolerance report, smoke, library rates at n = 50..64 on 888 custom units (a whole number of
# waves at 2 and at 3 blocks per SM), then the end-of-round evidence (tools/round_profile.sh).
set -u
O=gpurun_out/r02s12; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_wsplit.py -q > $O/pytest_wsplit.log 2>&1; echo "pytest_wsplit rc=$?" >> $O/status.txt
PERMB200_TOL_REPORT=$O/tol_report.json timeout 1500 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
for n in 50 51; do
  for alg in glynn ryser; do
    timeout 300 python tools/profile_sweep.py --custom 11,4,7 --units 888 --reps 3 --n $n --alg $alg >> $O/large_n.log 2>&1
  done
done
for n in 52 53 54 55 56 58 60 61 62 63 64; do
  for alg in glynn ryser; do
    [ "$n$alg" = "64ryser" ] && continue
    timeout 300 python tools/profile_sweep.py --custom 11,4,6 --units 888 --reps 3 --n $n --alg $alg >> $O/large_n.log 2>&1
  done
done
echo "large_n done" >> $O/status.txt
bash tools/round_profile.sh > $O/round_profile.log 2>&1; echo "round_profile rc=$?" >> $O/status.txt
echo "pre12 done $(date)" >> $O/status.txt
