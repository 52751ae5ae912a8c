"""Opcode mix of the largest fp64 basic blocks of one kernel in a cubin/.so (static, no GPU).

usage: python tools/sass_blocks.py lib.so mangled_kernel_name [n_blocks]
"""
import re
import subprocess
import sys
from collections import Counter

so, fn = sys.argv[1], sys.argv[2]
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 2
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, so], capture_output=True, text=True).stdout
ins = []
for line in sass.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
targets = set()
for _, t in ins:
    m = re.search(r"BRA(?:\.[A-Z.]+)? (?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
    if m and m.group(1):
        targets.add(int(m.group(1), 16))
blocks, cur = [], []
for addr, t in ins:
    if addr in targets and cur:
        blocks.append(cur)
        cur = []
    cur.append(t)
    if re.search(r"\bBRA\b|\bEXIT\b|\bRET\b", t):
        blocks.append(cur)
        cur = []
if cur:
    blocks.append(cur)
fp = [b for b in blocks if any(x.split()[0].startswith(("DFMA", "DADD", "DMUL")) or
                               (x.startswith("@") and x.split()[1].startswith(("DFMA", "DADD"))) for x in b)]
for b in sorted(fp, key=len, reverse=True)[:nb]:
    c = Counter((x.split()[1] if x.startswith("@") else x.split()[0]) for x in b)
    print(f"block of {len(b)} instructions:")
    for op, k in c.most_common():
        print(f"  {k:4d} {op}")
