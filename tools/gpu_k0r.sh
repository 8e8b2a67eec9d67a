# K0 floor rank (DTOPK_K0_R): filter fallback flags, then sweep A/B
for v in r125 r110 r103; do
  for k in 1048576 524288 65536; do
    DTOPK_LIB=paper_2109_08219_b200/_lib/var/lib_$v.so timeout 120 python tools/prof_case.py --k $k --reps 2 2>&1 | python -c "import sys,ast; l=sys.stdin.read().strip().splitlines()[-1]; d=ast.literal_eval(l[l.index('{'):]); print('$v', $k, 'filtered', d.get('filtered'), 'fallback', d.get('filter_fallback'))"
  done
done
EXPS=${EXPS:-16,18,19,20} bash tools/ab_variants.sh r125 r110 r103 r125 r110 r103 r125 r110 r103
