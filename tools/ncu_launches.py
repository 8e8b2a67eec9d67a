"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/ncu_launches.py gpurun_out/launches_k1024.csv [more.csv ...]

Prints, per file, the kernels of the last dtopk_select (from the last
k1_delegates launch on) with their serialised, cold-cache durations.
"""

import csv
import sys


def table(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    out = [(r[ki].split("(")[0].replace("void ", "")[:34], float(r[vi]) / 1000) for r in rows[start + 1:] if len(r) > vi]
    first = max(i for i, o in enumerate(out) if o[0].startswith("k1_delegates"))
    return out[first:]


if __name__ == "__main__":
    for path in sys.argv[1:]:
        t = table(path)
        total = sum(x for _, x in t)
        print(f"{path}: {len(t)} launches, {total:.1f} us")
        print("   " + "  ".join(f"{n}={x:.1f}" for n, x in t))
