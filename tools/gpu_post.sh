# After the round-end run: new pass-3 GPU tests, warm launch list at HEAD (k = 2^20, 2^14), sanitizer (quick set)
mkdir -p gpurun_out/post gpurun_out/post/sanitizer
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "pass3 or graph_plan or big_answer" > gpurun_out/post/gputest.log 2>&1; echo gputest_rc=$?; tail -3 gpurun_out/post/gputest.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for k in 1048576 16384; do
  timeout 300 ncu --metrics $M --cache-control none --clock-control none --csv --log-file gpurun_out/post/launches_k${k}_warm.csv \
    python tools/prof_case.py --k $k --reps 3 > /dev/null 2>&1
done
python tools/ncu_launches.py gpurun_out/post/launches_k*_warm.csv > gpurun_out/post/launches_warm.txt; cat gpurun_out/post/launches_warm.txt
CS=/usr/local/cuda/bin/compute-sanitizer; O=gpurun_out/post/sanitizer
timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_cases.py quick > $O/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/memcheck.log
timeout 1200 $CS --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize_cases.py quick > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/racecheck.log
timeout 900 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py quick > $O/synccheck.log 2>&1; echo "synccheck rc=$?" >> $O/synccheck.log
tail -n 4 $O/*.log
