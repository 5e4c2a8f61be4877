"""Builds profiles/ncu_traffic.json (read by bench.py for roofline.traffic) from
the per-config ncu DRAM captures of tools/prof_r2.sh:

    python tools/dram_traffic.py r2c      # reads gpurun_out/r2c_dram_config{0..4}.csv
"""
import csv
import io
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1]
LABEL = {"k_pa": "fx_explicit_sweep_r", "k_plane": "fx_plane_vy_update", "k_fx_explicit": "fx_explicit",
         "k_ex4": "fx_explicit", "k_fx_r": "fx_sweep_r", "k_fx_v": "fx_sweep_v", "k_y3": "fx_sweep_y_update",
         "k_fx_y": "fx_sweep_y_update"}
out = {"_note": f"DRAM bytes (read + write) per launch from `ncu --metrics dram__bytes_read.sum,"
                f"dram__bytes_write.sum,gpu__time_duration.sum` (tools/prof_r2.sh, build {R}, one B200; "
                "ncu flushes L2 before each replay), keyed by config and by the bench's kernel label; "
                "read by bench.py for roofline.traffic"}
for c in range(5):
    path = os.path.join(ROOT, "gpurun_out", f"{R}_dram_config{c}.csv")
    if not os.path.exists(path):
        continue
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = defaultdict(lambda: defaultdict(list))  # label -> metric -> values
    names = {}
    for r in rows:
        kn = r["Kernel Name"].split("::")[-1]
        base = kn.split("<")[0]
        lab = LABEL.get(base)
        if not lab:
            continue
        names[lab] = kn.split("(")[0]
        per[lab][r["Metric Name"]].append(float(r["Metric Value"].replace(",", "")))
    cfg = {}
    for lab, m in per.items():
        rd, wr = m.get("dram__bytes_read.sum", [0]), m.get("dram__bytes_write.sum", [0])
        t = m.get("gpu__time_duration.sum", [0])
        n = len(rd)
        cfg[lab] = {"kernel": names[lab], "launches": n, "dram_read_bytes": sum(rd) / n,
                    "dram_write_bytes": sum(wr) / len(wr), "dram_bytes": sum(rd) / n + sum(wr) / len(wr),
                    "duration_ns_cold": sum(t) / max(len(t), 1)}
    out[f"config{c}"] = cfg
with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({k: {l: round(v["dram_bytes"] / 1e6, 1) for l, v in c.items()} for k, c in out.items()
                  if k.startswith("config")}))
