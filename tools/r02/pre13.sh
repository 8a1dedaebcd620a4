#!/bin/bash
# Session 13: A/B of the 2-terms-per-iteration half-walk (PERMB200_UNROLL2_FROM; half the loop
# body, bit-identical results) against the 4-term loop: microbenchmarks (sweep_bench_u4 / _u2:
# n = 32..51 one lane; wsplit_bench_u2: n = 48..64, one lane with the 2-term loop vs the 2-lane
# and warp-pair splits), then the library built with the 2-term loop from n = 48
# and the 2-terms-per-exchange warp-pair walk (PERMB200_WSPLIT_U2)
# (libpermb200_u2.so, selected by PERMB200_LIB): M5 sample next to the default library's, the GPU
# suite, n = 50..56 rates, one ncu --set full capture of its sweep_kernel<50>.
set -u
O=gpurun_out/r02s13; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
for r in 1 2; do
  for v in u4 u2; do echo "== $v" >> $O/sweep_bench.log; timeout 600 tools/microbench/sweep_bench_$v 8 >> $O/sweep_bench.log 2>&1; done
done
echo "sweep_bench rc=$?" >> $O/status.txt
timeout 600 tools/microbench/wsplit_bench_u2 2 > $O/wsplit_bench_u2.log 2>&1; echo "wsplit_bench_u2 rc=$?" >> $O/status.txt
U2=$PWD/paper_1606_05836_b200/libpermb200_u2.so
timeout 600 python tools/perf_configs.py --skip M1,M2,M3,M4,DD --out $O/m5_default.json > $O/m5_default.log 2>&1; echo "m5_default rc=$?" >> $O/status.txt
PERMB200_LIB=$U2 timeout 600 python tools/perf_configs.py --skip M1,M2,M3,M4,DD --out $O/m5_u2.json > $O/m5_u2.log 2>&1; echo "m5_u2 rc=$?" >> $O/status.txt
PERMB200_LIB=$U2 PERMB200_TOL_REPORT=$O/tol_report_u2.json timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_u2.log 2>&1; echo "pytest_u2 rc=$?" >> $O/status.txt
for n in 48 49 50 51; do
  for alg in glynn ryser; do
    PERMB200_LIB=$U2 timeout 300 python tools/profile_sweep.py --custom 11,4,7 --units 888 --reps 3 --n $n --alg $alg >> $O/large_n_u2.log 2>&1
  done
done
for n in 52 54 56 58 60; do
  for alg in glynn ryser; do
    PERMB200_LIB=$U2 timeout 300 python tools/profile_sweep.py --custom 11,4,6 --units 888 --reps 3 --n $n --alg $alg >> $O/large_n_u2.log 2>&1
  done
done
echo "large_n_u2 done" >> $O/status.txt
P50="python tools/profile_sweep.py --workload M5 --custom 11,4,7 --units 296 --reps 1"
PERMB200_LIB=$U2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o $O/sweep_n50_u2 $P50 > $O/ncu50.log 2>&1; echo "ncu50 rc=$?" >> $O/status.txt
echo "pre13 done $(date)" >> $O/status.txt
