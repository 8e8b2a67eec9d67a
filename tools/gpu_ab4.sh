EXPS=${EXPS:-16,19,20} bash tools/ab_variants.sh base2 noopt base2 noopt base2 noopt
