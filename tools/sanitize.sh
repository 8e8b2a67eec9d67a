#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (run under gpurun); logs to $1.
O=${1:-gpurun_out/sanitize}
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_cases.py > $O/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/memcheck.log
timeout 1500 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py quick > $O/synccheck.log 2>&1; echo "synccheck rc=$?" >> $O/synccheck.log
timeout 2400 $CS --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize_cases.py quick > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/racecheck.log
tail -n 4 $O/*.log
