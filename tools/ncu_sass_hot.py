"""Top stalled SASS lines per kernel from `ncu --page source --csv --print-source sass`.

    python tools/ncu_sass_hot.py src.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
kern, hdr, lines = None, None, []


def flush():
    if kern and lines:
        tot = sum(s for s, _ in lines) or 1
        print(f"== {kern[:90]}  ({tot} samples)")
        for s, t in sorted(lines, reverse=True)[:top]:
            print(f"  {100.0 * s / tot:5.1f}%  {t}")


for r in rows:
    if r and r[0] == "Kernel Name":
        flush()
        kern, hdr, lines = r[1], None, []
    elif r and r[0] == "Address":
        hdr = r
    elif hdr and len(r) > 3:
        try:
            lines.append((int(r[2]), r[1].strip()))
        except ValueError:
            pass
flush()
