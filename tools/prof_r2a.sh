O=gpurun_out/r2a
mkdir -p $O
LAUNCH_KS="1024 65536 1048576" FULL_KS="1048576" bash tools/ncu_tail.sh $O > $O/tail.log 2>&1
for d in ascending few_distinct all_equal; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/launches_$d.csv python tools/prof_case.py --dist $d --k 65536 > $O/$d.out 2>&1
done
python tools/ncu_launches.py $O/launches_*.csv > $O/launches_summary.txt
