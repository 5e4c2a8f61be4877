"""Summarise an ncu source page (SASS view): top instructions by stall samples
and the shared-memory conflict hot spots.  python tools/ncu_hot.py rep [kernel-regex] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kern:
    cmd += ["-k", "regex:" + kern]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Address")
body = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
ix = {h: q for q, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(r, h):
    try:
        return float(r[ix[h]].replace(",", ""))
    except ValueError:
        return 0.0


tot = sum(num(r, "# Samples") for r in body) or 1.0
print(f"instructions={len(body)} samples={tot:.0f}")
agg = {h: sum(num(r, h) for r in body) for h in stalls}
print("stalls:", ", ".join(f"{h[6:]}={100 * v / tot:.1f}%" for h, v in sorted(agg.items(), key=lambda x: -x[1]) if v / tot > 0.01))
print("--- top instructions by samples")
for r in sorted(body, key=lambda r: -num(r, "# Samples"))[:N]:
    top = sorted(((num(r, h), h[6:]) for h in stalls), reverse=True)[:2]
    print(f"{r[ix['Address']][-5:]} {num(r, '# Samples'):6.0f} {r[ix['Source']].strip()[:60]:60s} "
          + " ".join(f"{n}={v:.0f}" for v, n in top if v))
print("--- shared excess wavefronts")
for r in sorted(body, key=lambda r: -num(r, "L1 Wavefronts Shared Excessive"))[:12]:
    if num(r, "L1 Wavefronts Shared Excessive") > 0:
        print(f"{r[ix['Address']][-5:]} excess={num(r, 'L1 Wavefronts Shared Excessive'):.0f} "
              f"ideal={num(r, 'L1 Wavefronts Shared Ideal'):.0f} {r[ix['Source']].strip()[:60]}")
