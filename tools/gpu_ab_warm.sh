mkdir -p gpurun_out/warm
export EXPS=12,14,15,17,19,20
bash tools/ab_variants.sh base p3s0 bkt1k bkt512 base p3s0 bkt1k bkt512 2>&1 | tee gpurun_out/ab/summary.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for k in 16384 1048576; do
  timeout 300 ncu --metrics $M --cache-control none --clock-control none --csv --log-file gpurun_out/warm/launches_k$k.csv \
    python tools/prof_case.py --k $k --reps 3 > /dev/null 2>&1
done
python tools/ncu_launches.py gpurun_out/warm/launches_*.csv | tee gpurun_out/warm/summary.txt
