#!/bin/bash
# Round profile set (run under gpurun): bench line, launch lists, K1 full ncu capture, configs 3-5.
#   bash tools/profile_round.sh r1
R=${1:-r1}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi -L > $O/gpu_info.txt; nproc >> $O/gpu_info.txt; lscpu | grep "Model name" >> $O/gpu_info.txt
timeout 600 python bench.py > $O/bench_full.json 2> $O/bench_full.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for k in 1024 65536 1048576; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_k$k.csv \
    python bench.py --k $k --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu --no-graph --no-sharded --no-configs > /dev/null 2>&1
done
python tools/ncu_launches.py $O/launches_k*.csv > $O/launches_summary.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1_delegates -s 3 -c 1 -o $O/k1_full \
  python bench.py --k 1024 --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu --no-graph --no-sharded --no-configs > /dev/null 2>&1
ncu -i $O/k1_full.ncu-rep --page raw --csv > $O/k1_delegates_ncu_full_raw.csv 2>/dev/null
timeout 400 python tools/bench_configs.py > $O/configs.json 2>&1
timeout 200 python tools/stage_times.py > $O/stage_times.txt 2>&1
ls -la $O
