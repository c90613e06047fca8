"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`.

  python tools/ncu_hotspots.py <src.csv> [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = next(r for r in rows if "Address" in r and "Source" in r)
start = rows.index(h) + 1
ai, si = h.index("Address"), h.index("Source")
wi = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[start:]:
    try:
        data.append((int(r[wi]), r[ai], r[si]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print(f"total stall samples {tot}")
for w, a, s in sorted(data, reverse=True)[:n]:
    print(f"{w:8d} {100 * w / tot:5.1f}%  {a[-6:]}  {s[:110]}")
