set -x
mkdir -p gpurun_out/p1
for k in 1024 8192 65536 1048576; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p1/launches_k$k.csv python bench.py --k $k --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu --no-graph > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1_delegates -s 3 -c 1 -o gpurun_out/p1/k1_full python bench.py --k 1024 --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu --no-graph > gpurun_out/p1/k1_full.log 2>&1
ls -la gpurun_out/p1
