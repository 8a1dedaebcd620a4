#!/bin/bash
# One time-limited GPU session of the measured Glynn-Ryser discrepancy ladder toward M5
# (VERDICT r01 item 3 fallback: full FP64 Glynn and Ryser permanents of synth.gaussian(n, 50) at
# n = 46 and 48, checkpointed): runs PRE, then the jobs in order, each resuming from
# runs/ladder/<job> (tracked in git) and mirroring its ledger + segment log (SM clocks) into
# gpurun_out/ladder/<job> after every segment, until TOTAL seconds after this script started.
#   bash tools/r02/ladder_session.sh <total_s> [pre-command]
set -u
T0=$(date +%s)
TOTAL=${1:-3300}
PRE=${2:-}
mkdir -p gpurun_out/ladder
if [ -n "$PRE" ]; then bash -c "$PRE"; fi
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv >> gpurun_out/ladder/smi.txt 2>&1
# LADDER_JOBS="41 glynn;41 ryser;..." overrides the job list (';'-separated "<n> <alg>" pairs)
IFS=';' read -ra JOBS <<< "${LADDER_JOBS:-46 glynn;46 ryser;48 glynn;48 ryser}"
for job in "${JOBS[@]}"; do
  set -- $job
  N=$1; ALG=$2; J=g${N}_${ALG}
  if [ -f runs/ladder/$J/COMPLETE ]; then continue; fi
  BUDGET=$(( TOTAL - ($(date +%s) - T0) - 240 ))
  [ $BUDGET -lt 90 ] && break
  # a job that cannot finish in what is left is skipped, not started (LADDER_NEED_<job> seconds)
  NEED_VAR=LADDER_NEED_${J}; NEED=${!NEED_VAR:-0}
  if [ $BUDGET -lt $NEED ]; then echo "$J skipped: budget $BUDGET < need $NEED" >> gpurun_out/ladder/session.log; continue; fi
  mkdir -p gpurun_out/ladder/$J runs/ladder/$J
  echo "$J start $(date) budget_s=$BUDGET" >> gpurun_out/ladder/session.log
  python tools/m5_run.py --workload gauss50:$N --alg $ALG --ledger-in runs/ladder/$J --out gpurun_out/ladder/$J \
      --budget-s $BUDGET >> gpurun_out/ladder/$J/session.log 2>&1
  echo "$J m5_run rc=$?" >> gpurun_out/ladder/session.log
  if grep -q '"complete": true' gpurun_out/ladder/$J/m5_status.json 2>/dev/null; then touch gpurun_out/ladder/$J/COMPLETE; fi
done
