EXPS=${EXPS:-17,19,20} bash tools/ab_variants.sh bk4 bk8 bk16 k2u8 bk4 bk8 bk16 k2u8 bk4 bk8 bk16 k2u8
