#!/bin/bash
# Local wrapper (runs HERE, not on the box): bring the previous sessions' Ryser ledgers from
# gpurun_out/m5r into runs/m5r (shipped with the snapshot), then one gpurun call that runs
# PRE and a Ryser session of BUDGET seconds.
#   bash tools/r02/launch_session.sh <pre-script> <budget_s> <timeout_s>
set -u
PRE=$1; BUDGET=$2; TO=$3
mkdir -p runs/m5r
for f in gpurun_out/m5r/m5_ryser.rank*.npz gpurun_out/m5r/segments.rank*.csv; do
  [ -e "$f" ] && cp -n "$f" runs/m5r/
done
ls runs/m5r | grep -c npz
exec /usr/local/graft/bin/gpurun --timeout $TO -- "bash tools/r02/ryser_session.sh $BUDGET \"bash $PRE\""
