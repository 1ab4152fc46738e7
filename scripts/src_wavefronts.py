"""Per-instruction shared-memory wavefronts and stall samples from an ncu
source-page export (--page source --csv --print-source sass): the top shared
accesses with their ideal wavefronts, and the stall reasons per opcode.

  python scripts/src_wavefronts.py src.csv [n_chunks]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_chunks = float(sys.argv[2]) if len(sys.argv) > 2 else 65536.0
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def v(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (ValueError, KeyError, IndexError):
        return 0.0


def op(r):
    t = r[ix["Source"]].split()
    return "" if not t else (t[1] if t[0].startswith("@") else t[0])


tw = sum(v(r, "L1 Wavefronts Shared") for r in data)
ti = sum(v(r, "Instructions Executed") for r in data)
print(f"per chunk: {ti / n_chunks:.0f} warp-instructions, {tw / n_chunks:.0f} shared wavefronts "
      f"(ideal {sum(v(r, 'L1 Wavefronts Shared Ideal') for r in data) / n_chunks:.0f})")
byop = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in data:
    o = op(r)
    byop[o][0] += v(r, "L1 Wavefronts Shared") / n_chunks
    byop[o][1] += v(r, "L1 Wavefronts Shared Ideal") / n_chunks
    byop[o][2] += v(r, "Instructions Executed") / n_chunks
print("shared wavefronts per chunk by opcode (actual / ideal / instr):")
for o, (a, b, c) in sorted(byop.items(), key=lambda x: -x[1][0])[:14]:
    if a > 0.5:
        print(f"  {o:28s} {a:7.1f} {b:7.1f} {c:7.1f}")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
per = collections.defaultdict(collections.Counter)
for r in data:
    o = op(r).split(".")[0]
    for s in stalls:
        x = v(r, s)
        tot[s] += x
        per[o][s] += x
T = sum(tot.values())
print("stall samples by opcode (top 12 opcodes, top reasons):")
for o, c in sorted(per.items(), key=lambda x: -sum(x[1].values()))[:12]:
    s = sum(c.values())
    print(f"  {o:10s} {100 * s / T:5.1f}%  " + ", ".join(f"{k[6:]} {100 * x / T:.1f}" for k, x in c.most_common(4)))
