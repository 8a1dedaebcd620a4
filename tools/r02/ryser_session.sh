#!/bin/bash
# One time-limited session of the full n = 50 Ryser permanent (M5, 2^50 Gray-code terms):
# resumes from runs/m5r (ledgers of the previous sessions), sweeps segments for BUDGET
# seconds, leaves this session's ledger + segment log (with SM clocks) in gpurun_out/m5r/.
#   bash tools/r02/ryser_session.sh <budget_s> [pre-command]
set -u
BUDGET=${1:-2400}
PRE=${2:-}
mkdir -p gpurun_out/m5r
if [ -n "$PRE" ]; then bash -c "$PRE"; fi
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv >> gpurun_out/m5r/smi.txt 2>&1
python tools/m5_run.py --alg ryser --ledger-in runs/m5r --out gpurun_out/m5r --budget-s $BUDGET \
    >> gpurun_out/m5r/session.log 2>&1
echo "m5_run rc=$?" >> gpurun_out/m5r/session.log
