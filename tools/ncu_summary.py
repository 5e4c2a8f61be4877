"""Markdown table of the headline metrics of every kernel in an ncu report.

usage: python tools/ncu_summary.py report.ncu-rep [nodes_per_launch]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nodes = float(sys.argv[2]) if len(sys.argv) > 2 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
M = [("duration us", "gpu__time_duration.sum", 1e-3), ("regs", "launch__registers_per_thread", 1),
     ("warp instr", "smsp__inst_executed.sum", 1), ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
     ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
     ("FP64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
     ("L1 %", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
     ("L2 %", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
     ("DRAM %", "dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
     ("DRAM read MB", "dram__bytes_read.sum", 1e-6), ("DRAM write MB", "dram__bytes_write.sum", 1e-6)]
print("| kernel | " + " | ".join(m[0] for m in M) + (" | thread-instr / node |" if nodes else " |"))
print("|---" * (len(M) + 1 + (1 if nodes else 0)) + "|")
for r in rows[2:]:
    d = dict(zip(hdr, r))
    vals = []
    for _, key, sc in M:
        v = d.get(key, "")
        try:
            x = float(v.replace(",", ""))
            unit = rows[1][hdr.index(key)]
            if key.startswith("dram__bytes") and unit in ("Mbyte", "MB"):
                x *= 1e6
            if key.startswith("dram__bytes") and unit in ("Gbyte", "GB"):
                x *= 1e9
            if key == "gpu__time_duration.sum" and unit in ("usecond", "us"):
                x *= 1e3
            vals.append(f"{x * sc:.1f}")
        except (ValueError, IndexError):
            vals.append(v)
    name = d.get("Kernel Name", "?").replace("void unnamed>::", "").split("(")[0]
    extra = ""
    if nodes:
        try:
            extra = f" | {float(d['smsp__inst_executed.sum']) * 32 / nodes:.0f}"
        except (KeyError, ValueError):
            extra = " | "
    print(f"| {name} | " + " | ".join(vals) + extra + " |")
