# K3 one-pass / bucket_sort gathers / pass-3 v2: marks, A/B (3 interleaved rounds), GPU tests, warm launch list
mkdir -p gpurun_out/ab gpurun_out/warm
DTOPK_LIB=paper_2109_08219_b200/_lib/var/lib_p3prof.so timeout 120 python tools/prof_case.py --k 1048576 --reps 3 2>&1 | grep -v "^uniform" | tail -2
EXPS=${EXPS:-14,17,18,19,20} bash tools/ab_variants.sh new2 all3 all3u2 new2 all3 all3u2 new2 all3 all3u2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/gputest.log 2>&1; echo gputest_rc=$?; tail -3 gpurun_out/ab/gputest.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 ncu --metrics $M --cache-control none --clock-control none --csv --log-file gpurun_out/warm/launches_k1048576_all3.csv \
    python tools/prof_case.py --k 1048576 --reps 3 > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/warm/launches_k1048576_all3.csv
