EXPS=${EXPS:-16,17,18,19,20} bash tools/ab_variants.sh r125 kb1m kb512k r125 kb1m kb512k r125 kb1m kb512k
