"""Tabulate tools/time_variants.sh-style output ("== <variant> rep k" headers, "<case>: X ms/call")."""
import collections
import re
import sys

d = collections.defaultdict(list)
order, v = [], None
for line in open(sys.argv[1]):
    m = re.match(r"== (\S+)", line)
    if m:
        v = m.group(1)
        if v not in order:
            order.append(v)
        continue
    m = re.match(r"(.*): ([\d.]+) ms/call", line)
    if m and v:
        d[(m.group(1), v)].append(float(m.group(2)))
cases = []
for (c, _) in d:
    if c not in cases:
        cases.append(c)
print(f"{'case (best of reps, ms)':48s}" + "".join(f"{x:>9s}" for x in order))
for c in cases:
    print(f"{c:48s}" + "".join(f"{min(d[(c, x)]):9.3f}" if (c, x) in d else f"{'-':>9s}" for x in order))
