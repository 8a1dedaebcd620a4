#!/bin/bash
# End-of-round evidence on one B200 (run from the repo root under gpurun):
#   1. bench.py line (no profiler)                     -> gpurun_out/final/bench_n1.json
#   2. ncu launch list of the same bench command        -> gpurun_out/final/bench_launches.csv
#   3. DRAM bytes of the bench's full sweep launch      -> gpurun_out/final/sweep_m4_dram.csv
#   4. ncu --set full of the M4 sweep (2048 units)      -> gpurun_out/final/sweep_n40_full.ncu-rep
#   5. per-config numbers                               -> gpurun_out/final/perf_configs.json
set -u
OUT=gpurun_out/final
mkdir -p $OUT
python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "bench rc=$?" > $OUT/status.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $OUT/bench_ncu.log 2>&1; echo "launches rc=$?" >> $OUT/status.txt
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:sweep_kernel -c 1 --csv --log-file $OUT/sweep_m4_dram.csv \
    python tools/profile_sweep.py --workload M4 --fraction 1 --reps 1 > $OUT/dram.log 2>&1; echo "dram rc=$?" >> $OUT/status.txt
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o $OUT/sweep_n40_full \
    python tools/profile_sweep.py --workload M4 --fraction 64 --reps 1 > $OUT/full.log 2>&1; echo "full rc=$?" >> $OUT/status.txt
timeout 900 python tools/perf_configs.py --out $OUT/perf_configs.json > $OUT/perf.log 2>&1; echo "perf rc=$?" >> $OUT/status.txt
