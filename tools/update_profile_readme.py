"""Refresh the measured numbers in profiles/README.md and the K1 ncu summary from
gpurun_out/r1 (after tools/profile_round.sh r1 ran under gpurun).

    python tools/update_profile_readme.py
"""
import csv
import json
import os
import re
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC, DST = os.path.join(ROOT, "gpurun_out", "r1"), os.path.join(ROOT, "profiles", "r1")
for f in ("bench_full.json", "bench_ref.json", "gpu_info.txt", "launches_k1024.csv", "launches_k65536.csv",
          "launches_k1048576.csv", "launches_summary.txt", "configs.json", "stage_times.txt", "config5_single_gpu.json"):
    shutil.copy(os.path.join(SRC, f), os.path.join(DST, f))
rows = list(csv.reader(open(os.path.join(SRC, "k1_delegates_ncu_full_raw.csv"))))
h = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes_read.sum.per_second",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]
with open(os.path.join(DST, "k1_delegates_ncu_full_raw.txt"), "w") as f:
    f.write("# ncu --set full --clock-control none, k1_delegates<0,2> (N=2^30 u32, alpha=11), one launch\n")
    for w in want:
        if w in h:
            i = h.index(w)
            f.write(f"{w:<70} {rows[2][i]:>16} {rows[1][i]}\n")
dram_pct = float(rows[2][h.index("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")])

p = os.path.join(ROOT, "profiles", "README.md")
s = open(p).read()
d = json.load(open(os.path.join(DST, "bench_full.json")))
sw = {x["k"]: x for x in d["k_sweep"]}
cfg = {c["case"]: c for c in (json.loads(l) for l in open(os.path.join(DST, "configs.json")) if l.startswith("{"))}
c5 = [json.loads(l) for l in open(os.path.join(DST, "config5_single_gpu.json")) if l.startswith("{")]
ref = json.load(open(os.path.join(DST, "bench_ref.json")))
row_k = [1, 16, 256, 1024, 4096, 16384, 65536, 262144, 524288, 1048576]
old = s[s.index("| k | 1 | 16 | 256"):s.index("`k_sweep_min_frac`")]
new = "| k | " + " | ".join(str(k) for k in row_k) + " |\n|" + "---|" * (len(row_k) + 1) + "\n"
new += "| ms | " + " | ".join(f"{sw[k]['ms']:.3f}" for k in row_k) + " |\n"
new += "| frac of peak | " + " | ".join(f"{sw[k]['frac_of_peak']:.2f}" for k in row_k) + " |\n\n"
s = s.replace(old, new)
r = d["roofline"]
subs = [
    (r"`k_sweep_min_frac` = [0-9.]+:", f"`k_sweep_min_frac` = {d['k_sweep_min_frac']:.3f}:"),
    (r"\| step \(CUDA-graph plan, input resident in HBM, 100 steps\) \| [0-9.]+ ms \|",
     f"| step (CUDA-graph plan, input resident in HBM, 100 steps) | {d['ms_per_step']:.3f} ms |"),
    (r"\| throughput \(`value`\) \| [0-9.e+]+ keys/s \|", f"| throughput (`value`) | {d['value'] / 1e12:.2f}e12 keys/s |"),
    (r"\| step roofline 4N / t \| [0-9.]+ TB/s = [0-9.]+ of measured peak \|",
     f"| step roofline 4N / t | {4 * 2**30 / d['ms_per_step'] / 1e9:.2f} TB/s = {r['step_frac']:.2f} of measured peak |"),
    (r"\| K1 `k1_delegates` live \(CUDA events on the launch stream, timed region\) \| [0-9.]+ ms → [0-9.]+ TB/s = [0-9.]+ of the copy peak \|",
     f"| K1 `k1_delegates` live (CUDA events on the launch stream, timed region) | {r['kernel_ms']:.3f} ms → {r['achieved'] / 1000:.2f} TB/s = {r['frac']:.2f} of the copy peak |"),
    (r"\| K1 ncu `gpu__dram_throughput` \| [0-9.]+ %", f"| K1 ncu `gpu__dram_throughput` | {dram_pct:.1f} %"),
    (r"\| e2e `dr_topk\(pinned host tensor\)` incl. the 4 GiB H2D \| [0-9.]+ ms",
     f"| e2e `dr_topk(pinned host tensor)` incl. the 4 GiB H2D | {d['e2e']['ms_per_step']:.1f} ms"),
    (r"\| `--impl reference` \(C oracle port partitioned, 16 threads, full 2\^30\) \| [0-9.e]+ keys/s \([0-9.]+ ms / step\) \|",
     f"| `--impl reference` (C oracle port partitioned, 16 threads, full 2^30) | {ref['value'] / 1e10:.2f}e10 keys/s ({ref['ms_per_step']:.1f} ms / step) |"),
]
for a, b in subs:
    s = re.sub(a, b, s)


def g(n):
    return cfg[n]


def tri(base):
    return (" / ".join(f"{g(f'{base} beta={b}')['ms']:.3f}" for b in (1, 2, 3)),
            " / ".join(f"{g(f'{base} beta={b}')['frac_of_peak']:.2f}" for b in (1, 2, 3)))


old = s[s.index("| f32 normal, beta 1 / 2 / 3, k=1024 |"):s.index("Ascending input is")]
nm, nf = tri("config3 normal_f32")
pm, pf = tri("config3 pareto_f32")
new = (f"| f32 normal, beta 1 / 2 / 3, k=1024 | {nm} | {nf} |\n| f32 Pareto, beta 1 / 2 / 3 | {pm} | {pf} |\n"
       + "".join(f"| {lab} | {g(c)['ms']:.3f} | {g(c)['frac_of_peak']:.2f} |\n" for lab, c in (
           ("ascending, k=2^16", "config4 ascending"), ("all-equal, k=2^16", "config4 all_equal"),
           ("few-distinct (16 values), k=2^16", "config4 few_distinct"),
           ("rint(N(1e8,10)) (~100 values), k=2^16", "config4 nd_u32")))
       + f"| N = 2^33 on one GPU, k = 2^10 / 2^20 | {c5[0]['ms']:.3f} / {c5[1]['ms']:.3f} | "
       f"{c5[0]['frac_of_peak']:.2f} / {c5[1]['frac_of_peak']:.2f} |\n\n")
s = s.replace(old, new)
s = re.sub(r"Changes this round, measured at k = 2\^20: 1.129 ms \(first profile\) → [0-9.]+ ms;",
           f"Changes this round, measured at k = 2^20: 1.129 ms (first profile) → {sw[1048576]['ms']:.3f} ms;", s)
s = re.sub(r"The GPU path is [0-9,]+x one host core and [0-9]+x the 16-thread port on device time",
           f"The GPU path is {d['value'] / d['cpu_baseline']['value']:,.0f}x one host core and "
           f"{d['value'] / ref['value']:.0f}x the 16-thread port on device time", s)
open(p, "w").write(s)
print(d["ms_per_step"], d["k_sweep_min_frac"])
