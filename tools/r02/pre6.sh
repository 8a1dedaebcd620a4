#!/bin/bash
# Session 6 pre-script: source-level ncu of the n = 50 sweep (the M5 kernel, FP64 pipe 0.855 vs
# 0.91 at n = 40), large-n rates (n = 50/51 one thread per chunk vs n = 52..64 two-lane split),
# and a compute-sanitizer probe (records whether the tool runs on this pool).
set -u
O=gpurun_out/r02s6; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/smi.txt 2>&1
P50G="python tools/profile_sweep.py --workload M5 --custom 11,4,7 --units 296 --reps 1"
$P50G > $O/plain_n50.log 2>&1; echo "plain50 rc=$?" > $O/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o $O/sweep_n50_glynn $P50G > $O/ncu50.log 2>&1; echo "ncu50 rc=$?" >> $O/status.txt
ncu -i $O/sweep_n50_glynn.ncu-rep --page source --csv > $O/n50_source.csv 2>&1
ncu -i $O/sweep_n50_glynn.ncu-rep --page raw --csv > $O/n50_raw.csv 2>&1
for n in 50 51 52 54 56 58 60 62 64; do
  for alg in glynn ryser; do
    wb=6; [ $n -le 51 ] && wb=7
    timeout 300 python tools/profile_sweep.py --custom 11,4,$wb --units 592 --reps 3 --n $n --alg $alg >> $O/large_n.log 2>&1
  done
done
echo "large_n done" >> $O/status.txt
for v in c0mb4 c1mb4 c0mb3 c0mb5 c1mb5 c0mb6 c0mb4 c1mb4 c0mb3 c0mb5 c1mb5 c0mb6; do
  echo "v $v" >> $O/batched_variants.log; timeout 120 tools/microbench/batched_bench_$v 4096 >> $O/batched_variants.log 2>&1
done
cat > /tmp/san_tiny.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, synth, paper_1606_05836_b200 as pb
A = torch.from_numpy(synth.gaussian(12, 1)).cuda()
print(complex(pb.glynn(A).item()), complex(pb.ryser(A).item()))
PY
timeout 300 compute-sanitizer --tool memcheck python /tmp/san_tiny.py > $O/sanitizer_probe.log 2>&1; echo "sanitizer rc=$?" >> $O/status.txt
echo "pre6 done $(date)" >> $O/status.txt
