"""Per-CUDA-line instruction counts and stall samples from an ncu report.
    python tools/ncu_lines.py rep kernel-regex [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
fname, hdr, rows = None, None, []
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit() and len(r) == len(hdr):
        rows.append((fname, r))
ix = {h: q for q, h in enumerate(hdr)}


def num(r, h):
    try:
        return float(r[ix[h]].replace(",", ""))
    except (ValueError, KeyError):
        return 0.0


tot_i = sum(num(r, "Instructions Executed") for _, r in rows) or 1
tot_s = sum(num(r, "# Samples") for _, r in rows) or 1
print(f"warp-instructions={tot_i:.0f} samples={tot_s:.0f}")
key = "# Samples" if len(sys.argv) > 4 else "Instructions Executed"
for f, r in sorted(rows, key=lambda x: -num(x[1], key))[:N]:
    print(f"{f}:{r[0]:>5} inst={100 * num(r, 'Instructions Executed') / tot_i:5.1f}% "
          f"samp={100 * num(r, '# Samples') / tot_s:5.1f}% | {r[1].strip()[:90]}")
