# pass-3 timing marks (DTOPK_P3_PROFILE variant) + A/B of the current build against base
mkdir -p gpurun_out/ab gpurun_out/p3
for k in 1048576 262144 16384; do
  DTOPK_LIB=paper_2109_08219_b200/_lib/var/lib_p3prof.so timeout 120 python tools/prof_case.py --k $k --reps 3 2>&1 | grep -v "^uniform" | tail -3
done
EXPS=${EXPS:-13,14,15,19,20} bash tools/ab_variants.sh base new2 new base new2 new
