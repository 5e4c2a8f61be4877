"""Opcode mix + stall samples per opcode from an `ncu --page source --csv --print-source sass` dump.

usage: python tools/sass_mix.py dump.csv [top]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
ix, isrc, ismp = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
inst, samp = Counter(), Counter()
for r in rows[2:]:
    if len(r) <= ix or not r[ix].strip().isdigit():
        continue
    op = r[isrc].split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    inst[o] += int(r[ix])
    samp[o] += int(r[ismp] or 0)
T, S = sum(inst.values()), sum(samp.values())
print(f"total warp-instr {T}  samples {S}")
for o, n in inst.most_common(top):
    print(f"{o:10s} {n:12d} {100*n/T:5.1f}%  stall-samples {100*samp[o]/S:5.1f}%")
