# K3 work units: GPU tests, sweep A/B, config-4 A/B
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/gputest.log 2>&1; echo gputest_rc=$?; tail -3 gpurun_out/ab/gputest.log
EXPS=${EXPS:-14,16,19,20} bash tools/ab_variants.sh base2 k3u base2 k3u
for v in base2 k3u base2 k3u; do
  DTOPK_LIB=paper_2109_08219_b200/_lib/var/lib_$v.so timeout 300 python bench.py --steps 50 --no-e2e --no-cpu --no-sharded --no-sweep --no-big > gpurun_out/ab/cfg_$v.json 2>/dev/null
  echo "== $v"; python tools/bench_summary.py gpurun_out/ab/cfg_$v.json | grep config
done
