#!/bin/bash
# Round-2 profile set (run under gpurun): bench lines, launch lists (uniform k = 2^10 / 2^16 / 2^20 and
# config 4), K1 ncu --set full captures (full mode, alpha 11; filtered mode, alpha 6), power-cap drift.
#   bash tools/profile_r2.sh gpurun_out/r2
O=${1:-gpurun_out/r2}
mkdir -p $O
nvidia-smi -L > $O/gpu_info.txt; nproc >> $O/gpu_info.txt; lscpu | grep "Model name" >> $O/gpu_info.txt
timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for k in 1024 65536 1048576; do
  timeout 300 ncu --metrics $M --clock-control none --csv --log-file $O/launches_k$k.csv \
    python tools/prof_case.py --k $k --reps 3 > /dev/null 2>&1
done
for d in ascending all_equal few_distinct; do
  timeout 300 ncu --metrics $M --clock-control none --csv --log-file $O/launches_$d.csv \
    python tools/prof_case.py --dist $d --k 65536 --reps 3 > /dev/null 2>&1
done
python tools/ncu_launches.py $O/launches_*.csv > $O/launches_summary.txt
for ks in 1024:1 1048576:2; do  # skip the first call's K1 (and, at 2^20, its flag-gated fallback launch)
  k=${ks%:*}; sk=${ks#*:}
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1_delegates -s $sk -c 1 -o $O/k1_k$k \
    python tools/prof_case.py --k $k --reps 2 > /dev/null 2>&1
  ncu -i $O/k1_k$k.ncu-rep --page raw --csv > $O/k1_k${k}_raw.csv 2>/dev/null
  rm -f $O/k1_k$k.ncu-rep
done
timeout 120 python tools/k1_drift.py > $O/k1_drift.txt 2>&1
ls -la $O
