# fast_tail phase clocks (DTOPK_FT_PROFILE variant) at the headline k and neighbours
for k in 1024 256 4096; do
  DTOPK_LIB=paper_2109_08219_b200/_lib/var/lib_ftprof.so timeout 120 python tools/prof_case.py --k $k --reps 3 2>&1 | grep -v "^uniform" | tail -2
done
