EXPS=${EXPS:-12,14,16,19,20} bash tools/ab_variants.sh c3 c3m3 c3 c3m3 c3 c3m3
