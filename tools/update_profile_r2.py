"""Copy the round-2 profile set (tools/profile_r2.sh under gpurun) into
profiles/r2 and write the K1 ncu summaries and a numbers table.

    python tools/update_profile_r2.py [gpurun_out/r2]
"""
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "r2")
DST = os.path.join(ROOT, "profiles", "r2")
os.makedirs(DST, exist_ok=True)
for f in os.listdir(SRC):
    if f.endswith((".json", ".txt")) or f.startswith("launches_"):
        shutil.copy(os.path.join(SRC, f), os.path.join(DST, f))

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes_read.sum.per_second",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]


def summarise(raw, out, title):
    rows = list(csv.reader(open(raw)))
    h = rows[0]
    with open(out, "w") as f:
        f.write(f"# ncu --set full --clock-control none, {title}, one launch\n")
        for w in WANT:
            if w in h:
                i = h.index(w)
                f.write(f"{w:<70} {rows[2][i]:>16} {rows[1][i]}\n")


for k, name, title in ((1024, "k1_delegates_ncu_full_raw.txt", "k1_delegates<0,2> (N=2^30 u32, k=1024, alpha=11, full mode)"),
                       (1048576, "k1_filtered_ncu_full_raw.txt",
                        "k1_delegates<0,2> (N=2^30 u32, k=2^20, alpha=6, filtered mode: records instead of D + meta)")):
    raw = os.path.join(SRC, f"k1_k{k}_raw.csv")
    if os.path.exists(raw):
        summarise(raw, os.path.join(DST, name), title)

b = json.loads(open(os.path.join(SRC, "bench_full.json")).read().splitlines()[-1])
lines = ["| quantity | value |", "|---|---|",
         f"| headline step (k = 1024, graph plan) | {b['ms_per_step']:.4f} ms = {b['value']:.3e} keys/s, "
         f"{b['roofline']['step_frac']:.3f} of the measured peak |",
         f"| K1 live (events, timed region) | {b['roofline']['kernel_ms']:.4f} ms -> {b['roofline']['achieved']:.0f} GB/s "
         f"= {b['roofline']['frac']:.3f} of the copy peak |",
         f"| k sweep minimum | {b['k_sweep_min_frac']:.3f} of the peak |",
         f"| e2e pinned host input | {b['e2e']['ms_per_step']:.1f} ms = {b['e2e']['pcie']['e2e_over_h2d']:.3f} x the pure "
         f"H2D ({b['e2e']['pcie']['h2d_gbs']:.1f} GB/s) |"]
if b["e2e"].get("numpy_input"):
    lines.append(f"| e2e numpy input | {b['e2e']['numpy_input']['ms_per_step']:.1f} ms |")
lines.append(f"| CPU baseline (1 core) | {b['cpu_baseline']['value']:.3e} keys/s |")
sweep = ["", "| k | " + " | ".join(str(s["k"]) for s in b["k_sweep"]) + " |",
         "|---|" + "---|" * len(b["k_sweep"]),
         "| ms | " + " | ".join(f"{s['ms']:.3f}" for s in b["k_sweep"]) + " |",
         "| frac | " + " | ".join(f"{s['frac_of_peak']:.2f}" for s in b["k_sweep"]) + " |"]
cfg = ["", "| case | ms | frac |", "|---|---|---|"] + [
    f"| {c['case']} | {c['ms']:.3f} | {c['frac_of_peak']:.2f} |" for c in b.get("configs", [])]
open(os.path.join(DST, "numbers.md"), "w").write("\n".join(lines + sweep + cfg) + "\n")
print("\n".join(lines + sweep + cfg))
