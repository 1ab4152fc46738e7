"""Per-source-line instruction and stall-sample totals from an ncu
`--page source --csv --print-source cuda,sass` dump."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
cur_file = None
out = []
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        n = int(float(r[7] or 0)); smp = int(float(r[4] or 0))
    except ValueError:
        continue
    out.append((n, smp, cur_file, r[0], r[1][:80]))
tot = sum(o[0] for o in out); tots = sum(o[1] for o in out)
print(f"total inst {tot:,} samples {tots:,}")
key = 0 if len(sys.argv) < 3 or sys.argv[2] == "inst" else 1
for o in sorted(out, key=lambda o: -o[key])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{o[0]:11,} {100*o[0]/tot:5.1f}%  smp {o[1]:6,} {100*o[1]/max(tots,1):5.1f}%  {o[2]}:{o[3]}  {o[4]}")
