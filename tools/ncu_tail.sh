#!/bin/bash
# Per-kernel ncu captures of the post-K1 chain (run under gpurun):
#   LAUNCH_KS="1024 65536" FULL_KS="1024" bash tools/ncu_tail.sh <outdir>
# LAUNCH_KS: launch list (gpu__time_duration + dram bytes, cold/serialised) of one eager dtopk_select per k.
# FULL_KS:   one `--set full` capture of every post-K1 kernel of one call per k, exported as raw / details csv
#            (the .ncu-rep itself is deleted: gpurun copies back at most 64 MiB).
O=${1:-gpurun_out/tail}
mkdir -p $O
RX=${RX:-'regex:^(fast|k2|k3|k4|k5|k6|finish|sort|bucket|merge|tail|scan|sel_|writeout)'}
for k in ${LAUNCH_KS-1024 1048576}; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $O/launches_k$k.csv \
    python bench.py --k $k --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu --no-graph --no-configs --no-sharded > /dev/null 2>&1
done
for k in ${FULL_KS-1024}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "$RX" -s 40 -c 40 -o $O/tail_k$k \
    python bench.py --k $k --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu --no-graph --no-configs --no-sharded > /dev/null 2>&1
  ncu -i $O/tail_k$k.ncu-rep --page raw --csv > $O/tail_k${k}_raw.csv 2>/dev/null
  ncu -i $O/tail_k$k.ncu-rep --page details --csv > $O/tail_k${k}_details.csv 2>/dev/null
  rm -f $O/tail_k$k.ncu-rep
done
ls -la $O
