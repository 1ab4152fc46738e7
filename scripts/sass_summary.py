"""Summarise an ncu source page (--print-source sass --csv): executed
instructions and stall samples per opcode, and the hottest instructions."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
by_op = collections.defaultdict(lambda: [0, 0])
hot = []
tot_i = tot_s = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    n = int(float(r[ix["Instructions Executed"]] or 0))
    smp = int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    by_op[op][0] += n
    by_op[op][1] += smp
    tot_i += n
    tot_s += smp
    hot.append((smp, n, r[ix["Address"]], src))
print(f"total inst {tot_i:,}  samples {tot_s:,}")
for op, (n, s) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{op:10s} inst {n:12,} ({100*n/max(tot_i,1):5.1f}%)  samples {s:8,} ({100*s/max(tot_s,1):5.1f}%)")
print("hottest:")
for smp, n, a, src in sorted(hot, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{smp:7,} {n:10,} {a} {src}")
