# A/B of library variants + GPU tests + a source-level ncu capture of k2_pass3 (k = 2^20)
mkdir -p gpurun_out/ab gpurun_out/p3
export EXPS=${EXPS:-12,13,14,15,16,20}
bash tools/ab_variants.sh ${VARIANTS:-base new bkfix base new bkfix}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/gputest.log 2>&1; echo gputest_rc=$?; tail -3 gpurun_out/ab/gputest.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k2_pass3 -s 1 -c 1 -o gpurun_out/p3/p3 \
  python tools/prof_case.py --k 1048576 --reps 2 > gpurun_out/p3/log.txt 2>&1
ncu -i gpurun_out/p3/p3.ncu-rep --page source --csv --print-source sass > gpurun_out/p3/p3_sass.csv 2>/dev/null
ncu -i gpurun_out/p3/p3.ncu-rep --page source --csv --print-source cuda > gpurun_out/p3/p3_cuda.csv 2>/dev/null
rm -f gpurun_out/p3/p3.ncu-rep; ls -la gpurun_out/p3
