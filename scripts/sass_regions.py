"""Summarise an ncu source-page export (SASS) of the decode kernel per code
region: warp-instructions and shared-memory wavefronts per 64-token chunk.

  ncu -i prof.ncu-rep --page source --csv --print-source sass > src.csv
  python scripts/sass_regions.py src.csv [n_chunks]
"""
import collections
import csv
import sys

path = sys.argv[1]
n_chunks = float(sys.argv[2]) if len(sys.argv) > 2 else 65536.0  # C2: 16 x 8 x 512
rows = list(csv.reader(open(path)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def val(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (ValueError, KeyError):
        return 0.0


def opcode(r):
    t = r[ix["Source"]].split()
    if not t:
        return ""
    return (t[1] if t[0].startswith("@") else t[0]).split(".")[0]


tot_i = sum(val(r, "Instructions Executed") for r in data) / n_chunks
tot_w = sum(val(r, "L1 Wavefronts Shared") for r in data) / n_chunks
print(f"warp-instructions per chunk {tot_i:.0f}; shared wavefronts per chunk {tot_w:.0f}")
ops = collections.Counter()
for r in data:
    ops[opcode(r)] += val(r, "Instructions Executed") / n_chunks
print("opcodes per chunk: " + ", ".join(f"{o} {c:.0f}" for o, c in ops.most_common(20)))
print()
print(f"{'first row':>9} {'instr/chunk':>11} {'wavefr/chunk':>12}  top opcodes")
B = 80
for b0 in range(0, len(data), B):
    blk = data[b0:b0 + B]
    ti = sum(val(r, "Instructions Executed") for r in blk) / n_chunks
    if ti < 5:
        continue
    tw = sum(val(r, "L1 Wavefronts Shared") for r in blk) / n_chunks
    c = collections.Counter()
    for r in blk:
        c[opcode(r)] += val(r, "Instructions Executed") / n_chunks
    print(f"{b0:9d} {ti:11.1f} {tw:12.1f}  " + " ".join(f"{o}:{v:.0f}" for o, v in c.most_common(7)))
