#!/bin/bash
# A/B library variants built by tools/build_variant.sh (bench.py lines into gpurun_out/ab/)
mkdir -p gpurun_out/ab
for v in "$@"; do
  DTOPK_LIB=paper_2109_08219_b200/_lib/var/lib_$v.so timeout 300 python bench.py --steps 50 --no-e2e --no-cpu --no-sharded --no-configs --sweep-stride ${STRIDE:-5} ${EXPS:+--sweep-exps $EXPS} > gpurun_out/ab/$v.json 2> gpurun_out/ab/$v.err
  python - "$v" <<'PY'
import json,sys
v=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/ab/{v}.json"))
    print(v, "ms", round(d["ms_per_step"],4), "k1_ms", round(d["roofline"]["kernel_ms"],4), "sweep", [(s["k"], s["ms"], round(s["stage_ms"]["Delegate"],4)) for s in d["k_sweep"]])
    print("   tail (ms - eager K1)", [(s["k"], round(s["ms"] - s["stage_ms"]["Delegate"], 4)) for s in d["k_sweep"]])
except Exception as e:
    print(v, "failed", e)
PY
done
