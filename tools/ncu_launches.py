"""Summarise an `ncu --metrics gpu__time_duration.sum[,dram__bytes_*] --csv` launch list.

    python tools/ncu_launches.py gpurun_out/launches_k1024.csv [more.csv ...]

Prints, per file, the kernels of the last dtopk_select (from the last
k1_delegates launch on) with their serialised, cold-cache durations (us) and,
when captured, DRAM bytes read + written (MB).
"""

import csv
import sys


def table(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ii = hdr.index("ID")
    launches = {}
    order = []
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        lid = r[ii]
        if lid not in launches:
            launches[lid] = {"name": r[ki].split("(")[0].replace("void ", "")[:34]}
            order.append(lid)
        launches[lid][r[mi]] = float(r[vi].replace(",", ""))
    out = [launches[i] for i in order]
    starts = [i for i, o in enumerate(out) if o["name"].startswith("k0_sample")] or \
        [i for i, o in enumerate(out) if o["name"].startswith("k1_delegates")]
    first = max(starts)
    return out[first:]


def fmt(o):
    t = o.get("gpu__time_duration.sum", 0.0) / 1000.0
    b = (o.get("dram__bytes_read.sum", 0.0) + o.get("dram__bytes_write.sum", 0.0)) / 1e6
    return f"{o['name']}={t:.1f}" + (f"/{b:.2f}MB" if "dram__bytes_read.sum" in o else "")


if __name__ == "__main__":
    for path in sys.argv[1:]:
        t = table(path)
        total = sum(o.get("gpu__time_duration.sum", 0.0) for o in t) / 1000.0
        print(f"{path}: {len(t)} launches, {total:.1f} us")
        print("   " + "  ".join(fmt(o) for o in t))
