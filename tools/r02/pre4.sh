set -u
O=gpurun_out/r02e; mkdir -p $O
PERMB200_TOL_REPORT=$O/tol_report.json timeout 1800 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" > $O/status.txt
timeout 300 python tools/r02/m1_plans.py > $O/m1_plans_glynn.log 2>&1; echo "m1g rc=$?" >> $O/status.txt
timeout 300 python tools/r02/m1_plans.py --alg ryser > $O/m1_plans_ryser.log 2>&1; echo "m1r rc=$?" >> $O/status.txt
timeout 300 python tools/latency_probe.py > $O/latency.log 2>&1; echo "latency rc=$?" >> $O/status.txt
for v in c0mb4 c1mb4 c1mb3 c0mb3 mb5 mb6 c0mb4 c1mb4 c1mb3 c0mb3 mb5 mb6; do echo "v $v" >> $O/batched_variants.log; timeout 120 tools/microbench/batched_bench_$v 4096 >> $O/batched_variants.log 2>&1; done
for n in 52 56 60 64; do for alg in glynn glynn_plain; do timeout 300 python tools/profile_sweep.py --custom 11,4,6 --units 592 --reps 3 --n $n --alg $alg >> $O/large_n.log 2>&1; done; done
bash tools/r02/sanitize.sh; cp -r gpurun_out/r02_sanitize $O/ 2>/dev/null
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --cache-control all -k regex:sweep_kernel -c 1 --csv --log-file $O/sweep_m4_traffic.csv python tools/profile_sweep.py --workload M4 --fraction 1 --reps 1 > $O/traffic.log 2>&1; echo "traffic rc=$?" >> $O/status.txt
