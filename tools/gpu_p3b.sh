# new pass 3: timing marks, A/B against the previous build, GPU tests; source-level ncu of the k = 2^20 tail kernels
mkdir -p gpurun_out/ab gpurun_out/src
for k in 1048576 262144 16384; do
  DTOPK_LIB=paper_2109_08219_b200/_lib/var/lib_p3prof.so timeout 120 python tools/prof_case.py --k $k --reps 3 2>&1 | grep -v "^uniform" | tail -3
done
EXPS=${EXPS:-12,14,16,18,19,20} bash tools/ab_variants.sh new2 p3new new2 p3new
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/gputest.log 2>&1; echo gputest_rc=$?; tail -3 gpurun_out/ab/gputest.log
for kn in bucket_sort k5_emit k3_classify; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$kn -s 1 -c 1 -o gpurun_out/src/$kn \
    python tools/prof_case.py --k 1048576 --reps 2 > gpurun_out/src/$kn.log 2>&1
  ncu -i gpurun_out/src/$kn.ncu-rep --page source --csv --print-source sass > gpurun_out/src/${kn}_sass.csv 2>/dev/null
  rm -f gpurun_out/src/$kn.ncu-rep
done
ls -la gpurun_out/src
