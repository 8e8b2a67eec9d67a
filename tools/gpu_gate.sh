# K2c/K2b behind a graph conditional: new graph tests, full GPU suite, A/B against the previous build
mkdir -p gpurun_out/ab
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "graph_plan" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/gputest.log 2>&1; echo gputest_rc=$?; tail -3 gpurun_out/ab/gputest.log
EXPS=${EXPS:-14,16,19,20} bash tools/ab_variants.sh base2 gate base2 gate base2 gate
timeout 300 python bench.py --steps 50 --no-e2e --no-cpu --no-sharded --no-sweep > gpurun_out/ab/configs_gate.json 2>/dev/null; python tools/bench_summary.py gpurun_out/ab/configs_gate.json | tail -12
