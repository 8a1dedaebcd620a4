#!/bin/bash
# One time-limited session of the full n = 50 Ryser permanent (M5, 2^50 Gray-code terms):
# runs PRE, then resumes from runs/m5r (ledgers of the previous sessions, tracked in git) and
# sweeps segments until TOTAL seconds after this script started (minus a margin for the final
# copy), leaving this session's ledger + segment log (with SM clocks) in gpurun_out/m5r/.
#   bash tools/r02/ryser_session.sh <total_s> [pre-command]
set -u
T0=$(date +%s)
TOTAL=${1:-2400}
PRE=${2:-}
mkdir -p gpurun_out/m5r
if [ -n "$PRE" ]; then bash -c "$PRE"; fi
BUDGET=$(( TOTAL - ($(date +%s) - T0) - 240 ))
echo "session start $(date) budget_s=$BUDGET" >> gpurun_out/m5r/session.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv >> gpurun_out/m5r/smi.txt 2>&1
if [ $BUDGET -gt 120 ]; then
  python tools/m5_run.py --alg ryser --ledger-in runs/m5r --out gpurun_out/m5r --budget-s $BUDGET \
      >> gpurun_out/m5r/session.log 2>&1
  echo "m5_run rc=$?" >> gpurun_out/m5r/session.log
fi
