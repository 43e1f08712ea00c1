"""Opcode histogram (weighted by executed warp instructions) and top stall
lines from an ncu --page source --csv --print-source sass dump."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ops = collections.Counter()
stalls = []
total = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    n = int(float(r[ix["Instructions Executed"]] or 0))
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += n
    total += n
    stalls.append((int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), src[:80], n))
print("total warp instructions:", total)
for op, n in ops.most_common(30):
    print(f"{op:12s} {n:12d} {100*n/total:6.2f}%")
print("--- top stall-sampled instructions")
for s, src, n in sorted(stalls, reverse=True)[:25]:
    print(f"{s:7d} {n:10d}  {src}")
