#!/bin/bash
# ncu launch lists (serialised, cold cache) of library variants: tools/ab_launches.sh "k1 k2" v1 v2 ...
mkdir -p gpurun_out/abl
ks=$1; shift
for v in "$@"; do
  for k in $ks; do
    DTOPK_LIB=paper_2109_08219_b200/_lib/var/lib_$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/abl/${v}_k$k.csv python bench.py --k $k --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu --no-graph > /dev/null 2>&1
    python tools/ncu_launches.py gpurun_out/abl/${v}_k$k.csv
  done
done
