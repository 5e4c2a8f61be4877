"""Samples and instructions between barrier-like instructions of a kernel, in SASS address order:
    python tools/ncu_phases.py rep kernel-regex
A coarse phase profile of a straight-line kernel (phases are separated by BAR / UCGABAR / WARPSYNC)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: q for q, h in enumerate(hdr)}
body, seen = [], set()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) == len(hdr) and r[0] not in seen:
        seen.add(r[0]); body.append(r)
def num(r, h):
    try: return float(r[ix[h]].replace(",", ""))
    except ValueError: return 0.0
tot_s = sum(num(r, "# Samples") for r in body) or 1
tot_i = sum(num(r, "Instructions Executed") for r in body) or 1
acc_s = acc_i = 0.0; n = 0; first = body[0][0][-5:]
marks = ("BAR.SYNC", "UCGABAR_WAIT", "BAR.ARV", "EXIT")
for r in body:
    acc_s += num(r, "# Samples"); acc_i += num(r, "Instructions Executed"); n += 1
    src = r[ix["Source"]]
    if any(m in src for m in marks):
        if acc_s / tot_s > 0.002:
            print(f"{first}..{r[0][-5:]} {n:5d} sass  inst {100*acc_i/tot_i:5.1f}%  samples {100*acc_s/tot_s:5.1f}%   ends at {src.strip()[:40]}")
        acc_s = acc_i = 0.0; n = 0; first = r[0][-5:]
