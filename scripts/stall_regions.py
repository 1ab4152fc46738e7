"""Stall-reason samples per code region from an ncu source-page (SASS) CSV.

  python scripts/stall_regions.py src.csv [region_size]
Prints the total stall mix and, per region of `region_size` SASS rows, the
share of all samples and its top stall reasons.
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
size = int(sys.argv[2]) if len(sys.argv) > 2 else 80
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (ValueError, KeyError):
        return 0.0


tot = defaultdict(float)
reg = defaultdict(lambda: defaultdict(float))
for n, r in enumerate(data):
    for k in reasons:
        v = f(r, k)
        tot[k] += v
        reg[n // size][k] += v
T = sum(tot.values()) or 1.0
print("total:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]))
for g in sorted(reg):
    s = sum(reg[g].values())
    if s / T < 0.01:
        continue
    top = sorted(reg[g].items(), key=lambda x: -x[1])[:5]
    print(f"{g * size:6d} {100 * s / T:5.1f}%  " + " ".join(f"{k[6:]}:{100 * v / T:.1f}" for k, v in top))
