# pass 3 v2: timing marks, A/B (3 interleaved rounds), GPU tests
mkdir -p gpurun_out/ab
for k in 1048576 524288 16384; do
  DTOPK_LIB=paper_2109_08219_b200/_lib/var/lib_p3prof.so timeout 120 python tools/prof_case.py --k $k --reps 3 2>&1 | grep -v "^uniform" | tail -2
done
EXPS=${EXPS:-14,17,18,19,20} bash tools/ab_variants.sh new2 p3new2 new2 p3new2 new2 p3new2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/gputest.log 2>&1; echo gputest_rc=$?; tail -3 gpurun_out/ab/gputest.log
