#!/usr/bin/env python
"""Per-kernel stall breakdown and hottest SASS lines from `ncu --page source --csv`."""
import csv
import sys
from collections import Counter


def num(x):
    try:
        return float(x or 0)
    except ValueError:
        return None


rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h) and num(r[h.index("# Samples")]) is not None]
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = Counter()
for d in data:
    for c in stall_cols:
        tot[c] += num(d[c]) or 0
s = sum(tot.values())
print("stall reasons (all samples):")
for c, v in tot.most_common(10):
    print(f"  {c:28s} {100 * v / max(s, 1):5.1f} %")
key = "Warp Stall Sampling (All Samples)"
top = sorted(data, key=lambda d: -(num(d.get(key)) or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]
print("hottest instructions:")
for d in top:
    st = sorted(((num(d[c]) or 0, c) for c in stall_cols), reverse=True)[:2]
    print(f"  {d[key]:>6} {d['Source'][:70]:70s} {st[0][1]}={st[0][0]:.0f} {st[1][1]}={st[1][0]:.0f}")
