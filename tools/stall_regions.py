"""Stall reasons per address region of an `ncu --page source --csv --print-source sass` dump.

usage: python tools/stall_regions.py dump.csv start:end[:name] ...   (hex offsets from the kernel start)
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, iex = hdr.index("Address"), hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in reasons}
data = []
for r in rows[2:]:
    if len(r) <= iex or not r[iex].isdigit():
        continue
    data.append((int(r[ia], 16), int(r[iex]), {h: int(r[idx[h]] or 0) for h in reasons}))
base = data[0][0]
tot_s = sum(sum(d[2].values()) for d in data)
tot_i = sum(d[1] for d in data)
for spec in sys.argv[2:]:
    parts = spec.split(":")
    lo, hi = int(parts[0], 16), int(parts[1], 16)
    name = parts[2] if len(parts) > 2 else spec
    c, ni = Counter(), 0
    for a, e, st in data:
        if lo <= a - base < hi:
            c.update(st)
            ni += e
    n = sum(c.values()) or 1
    print(f"{name}: {100 * ni / tot_i:.1f}% instr, {100 * n / tot_s:.1f}% samples; " +
          ", ".join(f"{k[6:]} {100 * v / n:.0f}%" for k, v in c.most_common(8)))
