"""Dev tool: top stall-sampled SASS lines of an `ncu --page source --csv --print-source sass` dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    try:
        data.append((float(r[ci["Warp Stall Sampling (All Samples)"]] or 0), r[ci["Address"]], r[ci["Source"]].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0] / tot * 100:5.1f}% {d[1][-5:]} {d[2][:100]}")
