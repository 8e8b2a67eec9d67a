"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`.

    ncu -i rep --page source --csv --kernel-name K --print-source sass > k.csv
    python tools/ncu_sass_top.py k.csv [N]
"""
import csv
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]
si, ii, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
stallcols = [i for i, name in enumerate(h) if name.startswith("stall_")]
tot = sum(f(r[si]) for r in data)
print("samples", tot, "warp instrs", sum(f(r[ii]) for r in data), "sass lines", len(data))
agg = {}
for r in data:
    for i in stallcols:
        agg[h[i]] = agg.get(h[i], 0) + f(r[i])
print("stall totals:", sorted(((round(v), k) for k, v in agg.items()), reverse=True)[:8])
for r in sorted(data, key=lambda r: -f(r[si]))[:n]:
    st = sorted(((f(r[i]), h[i][6:]) for i in stallcols), reverse=True)[:2]
    print(r[0], r[src][:64].ljust(64), int(f(r[si])), int(f(r[ii])), st)
