EXPS=${EXPS:-10,14,16,19,20} bash tools/ab_variants.sh r125 cps2 cps3 cps5 r125 cps2 cps3 cps5 r125 cps2 cps3 cps5
