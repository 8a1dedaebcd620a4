#!/bin/bash
# Session 11 pre-script: the warp-pair row split (perm_kernels_wsplit.cuh) -- A/B against the
# one-lane sweep and the 2-lane split (wsplit_bench), library rates at n = 50..64 on the same
# custom units as profiles/r02_large_n_rates.log, its parity tests, the full GPU suite, and one
# ncu --set full capture of wsplit_kernel<52>.
set -u
O=gpurun_out/r02s11; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
for r in 1 2; do timeout 600 tools/microbench/wsplit_bench 2 >> $O/wsplit_bench.log 2>&1; done
echo "bench rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests/test_gpu_wsplit.py -x -q > $O/pytest_wsplit.log 2>&1; echo "pytest_wsplit rc=$?" >> $O/status.txt
for n in 52 53 54 56 58 60 62 64; do
  for alg in glynn ryser; do
    timeout 300 python tools/profile_sweep.py --custom 11,4,6 --units 592 --reps 3 --n $n --alg $alg >> $O/large_n.log 2>&1
  done
done
echo "large_n done" >> $O/status.txt
PERMB200_TOL_REPORT=$O/tol_report.json timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
P52="python tools/profile_sweep.py --n 52 --custom 11,4,6 --units 444 --reps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wsplit_kernel -c 1 -o $O/wsplit_n52 $P52 > $O/ncu52.log 2>&1; echo "ncu52 rc=$?" >> $O/status.txt
ncu -i $O/wsplit_n52.ncu-rep --page raw --csv > $O/n52_raw.csv 2>&1
ncu -i $O/wsplit_n52.ncu-rep --page source --csv > $O/n52_source.csv 2>&1
echo "pre11 done $(date)" >> $O/status.txt
