"""Print the headline, k sweep and config rows of a bench.py JSON line (compact).

    python tools/bench_summary.py gpurun_out/r2b/bench_full.json
"""
import json
import sys

d = json.loads([ln for ln in open(sys.argv[1]) if ln.startswith("{")][-1])
print("headline ms", round(d["ms_per_step"], 4), "frac", round(d["roofline"]["frac"], 3), "clocks", d.get("clocks"))
print("k_sweep_min_frac", round(d.get("k_sweep_min_frac", 0), 4))
for r in d.get("k_sweep", []):
    print(" k", r["k"], "a", r["alpha"], r["ms"], round(r["frac_of_peak"], 3), r.get("stage_ms"))
for r in d.get("configs", []):
    print(" ", r["case"], r["ms"], round(r["frac_of_peak"], 3))
