"""Opcode mix + hottest basic blocks from an ncu source page (--page source --csv --print-source sass)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[1], rows[2:]
ia, isrc, iss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
n = lambda r: int(r[ia]) if r[ia].isdigit() else 0
tot = sum(n(r) for r in data)
print("total warp instructions", tot)
c, st = Counter(), Counter()
for r in data:
    t = r[isrc].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    c[op.split(".")[0]] += n(r)
    st[op.split(".")[0]] += int(r[iss] or 0)
for op, k in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{op:10s} {k:12d} {k / tot * 100:5.1f}%  stall-samples {st[op]}")
# basic blocks = runs of equal execution count
blocks, i = [], 0
while i < len(data):
    j = i
    while j + 1 < len(data) and n(data[j + 1]) == n(data[i]):
        j += 1
    blocks.append((n(data[i]) * (j - i + 1), i, j))
    i = j + 1
print("--- hottest blocks (share of instructions, rows, count x len)")
for w, i, j in sorted(blocks, reverse=True)[:12]:
    print(f"{w / tot * 100:5.1f}%  rows {i}-{j}  {n(data[i])} x {j - i + 1}")
