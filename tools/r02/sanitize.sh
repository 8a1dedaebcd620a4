#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/r02/sanitize_cases.py, each after
# a clean plain run of the same command.  Summaries -> gpurun_out/r02_sanitize/.
set -u
O=gpurun_out/r02_sanitize; mkdir -p $O
timeout 600 python tools/r02/sanitize_cases.py > $O/plain.log 2>&1; echo "plain rc=$?" > $O/status.txt
timeout 1200 compute-sanitizer --tool memcheck --leak-check full python tools/r02/sanitize_cases.py > $O/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/status.txt
timeout 600 python tools/r02/sanitize_cases.py --small > $O/plain_small.log 2>&1; echo "plain_small rc=$?" >> $O/status.txt
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report all python tools/r02/sanitize_cases.py --small > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/status.txt
timeout 1200 compute-sanitizer --tool synccheck python tools/r02/sanitize_cases.py --small > $O/synccheck.log 2>&1; echo "synccheck rc=$?" >> $O/status.txt
