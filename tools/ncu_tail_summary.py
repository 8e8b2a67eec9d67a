"""Summarise an ncu --set full raw CSV of the post-K1 kernels (tools/prof_tail.sh):
per launch the duration, DRAM bytes, grid, registers, achieved occupancy, the
busiest / average SM active cycles (a max far above the average = one CTA's
serial tail) and the top three stall reasons.

    python tools/ncu_tail_summary.py gpurun_out/r2b/tail_uniform_k1048576_raw.csv > profiles/r2/tail_....txt
"""
import csv
import sys

STALLS = ["long_scoreboard", "short_scoreboard", "barrier", "no_instruction", "wait", "lg_throttle", "membar",
          "branch_resolving", "mio_throttle", "math_pipe_throttle", "drain", "not_selected", "dispatch_stall"]


UNITS = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def mbytes(units, h, r, n):
    if n not in h:
        return 0.0
    i = h.index(n)
    return float(r[i]) * UNITS.get(units[i], 1e-6)


def main(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]

    def g(r, n, default="-"):
        return r[h.index(n)] if n in h else default

    print(f"# {path.split('/')[-1]}: ncu --set full --clock-control none (cold caches, serialised launches)")
    print(f"{'kernel':<34} {'us':>7} {'rd MB':>8} {'wr MB':>7} {'grid':>5} {'regs':>4} {'occ%':>5} "
          f"{'smact avg':>9} {'smact max':>9}  top stalls (cycles per issue)")
    for r in rows[2:]:
        name = g(r, "Kernel Name").replace("void ", "").split("(")[0][:34]
        st = []
        for s in STALLS:
            v = g(r, f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio", "0")
            try:
                st.append((float(v), s))
            except ValueError:
                pass
        st.sort(reverse=True)
        top = ", ".join(f"{s} {v:.1f}" for v, s in st[:3])
        rd = mbytes(rows[1], h, r, "dram__bytes_read.sum")
        wr = mbytes(rows[1], h, r, "dram__bytes_write.sum")
        print(f"{name:<34} {float(g(r, 'gpu__time_duration.sum', '0')):>7.1f} "
              f"{rd:>8.2f} {wr:>7.2f} {g(r, 'launch__grid_size'):>5} {g(r, 'launch__registers_per_thread'):>4} "
              f"{float(g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active', '0')):>5.1f} "
              f"{float(g(r, 'sm__cycles_active.avg', '0')):>9.0f} {float(g(r, 'sm__cycles_active.max', '0')):>9.0f}  {top}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
