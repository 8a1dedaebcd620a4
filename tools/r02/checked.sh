#!/bin/bash
# Substitute for compute-sanitizer (closed on this pool): the bounds-checked build of the library
# (device-side checks of every shared-memory / table index, trap on failure) over the sanitizer
# cases and the whole GPU parity suite, plus the determinism stress as a race-detector proxy.
set -u
O=gpurun_out/r02_checked; mkdir -p $O
L=$PWD/paper_1606_05836_b200/libpermb200_checked.so
PERMB200_LIB=$L timeout 600 python tools/r02/sanitize_cases.py > $O/cases.log 2>&1; echo "checked cases rc=$?" > $O/status.txt
PERMB200_LIB=$L timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/pytest_checked.log 2>&1; echo "checked pytest rc=$?" >> $O/status.txt
timeout 900 python tools/r02/determinism.py --reps 100 > $O/determinism.log 2>&1; echo "determinism rc=$?" >> $O/status.txt
