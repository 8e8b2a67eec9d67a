# Final verification at HEAD: GPU tests + smoke + a short bench line
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-sharded --no-configs --sweep-stride 4 > gpurun_out/verify_bench.json 2>/dev/null; python tools/bench_summary.py gpurun_out/verify_bench.json
