# Round check under gpurun: GPU tests, the bench line, ncu --set full captures of the post-K1 kernels.
#   bash tools/gpu_round_check.sh [notests]
set -x
O=gpurun_out/r2b
mkdir -p $O
nvidia-smi -L
if [ "$1" != notests ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo gputest_rc=$?
  tail -5 $O/gputest.log
fi
timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err; echo bench_rc=$?
python tools/bench_summary.py $O/bench_full.json
bash tools/prof_tail.sh $O 1048576 uniform
bash tools/prof_tail.sh $O 65536 ascending
ls -la $O
