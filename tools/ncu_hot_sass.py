"""Top warp-stall SASS lines of one kernel from `ncu -i X.ncu-rep --page source --csv` output.

    ncu -i X.ncu-rep --page source --csv -k regex:NAME > /tmp/src.csv; python tools/ncu_hot_sass.py /tmp/src.csv [n]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
k = ci["Warp Stall Sampling (All Samples)"]
data = []
for r in rows[2:]:
    try:
        data.append((float(r[k]), r[ci["Address"]][-5:], r[ci["Source"]].strip()[:100]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1.0
for v, a, s in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v / tot * 100:5.1f}%  {a}  {s}")
