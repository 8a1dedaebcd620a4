#!/bin/bash
# Local wrapper (runs HERE, not on the box): bring the previous sessions' Ryser ledgers from
# gpurun_out/m5r into runs/m5r (tracked in git, shipped with the snapshot), then one gpurun call
# that runs PRE and a Ryser session filling TOTAL seconds; the gpurun timeout leaves a margin.
#   bash tools/r02/launch_session.sh <pre-script|-> <total_s>
set -u
PRE=$1; TOTAL=$2
mkdir -p runs/m5r
for f in gpurun_out/m5r/m5_ryser.rank*.npz gpurun_out/m5r/segments.rank*.csv; do
  [ -e "$f" ] && cp -n "$f" runs/m5r/
done
ls runs/m5r | grep -c npz
P=""; [ "$PRE" != "-" ] && P="bash $PRE"
TO=$((TOTAL + 300)); [ $TO -gt 3600 ] && TO=3600   # gpurun clamps a call to 3600 s
exec /usr/local/graft/bin/gpurun --timeout $TO -- "bash tools/r02/ryser_session.sh $TOTAL \"$P\""
