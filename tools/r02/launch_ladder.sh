#!/bin/bash
# Local wrapper (runs HERE): bring the previous sessions' ladder ledgers from gpurun_out/ladder
# into runs/ladder (tracked in git, shipped with the snapshot), then one gpurun call running PRE
# and a ladder session filling TOTAL seconds (gpurun clamps a call to 3600 s).
#   bash tools/r02/launch_ladder.sh <pre-script|-> <total_s>
set -u
PRE=$1; TOTAL=$2
for d in gpurun_out/ladder/g*; do
  [ -d "$d" ] || continue
  J=$(basename $d); mkdir -p runs/ladder/$J
  for f in $d/m5_*.rank*.npz $d/segments.rank*.csv $d/m5_status.json $d/COMPLETE; do
    [ -e "$f" ] && cp "$f" runs/ladder/$J/
  done
done
ls runs/ladder 2>/dev/null
P=""; [ "$PRE" != "-" ] && P="bash $PRE"
TO=$((TOTAL + 300)); [ $TO -gt 3600 ] && TO=3600
exec /usr/local/graft/bin/gpurun --timeout $TO -- "bash tools/r02/ladder_session.sh $TOTAL \"$P\""
