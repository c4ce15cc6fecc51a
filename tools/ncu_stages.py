"""Per-launch summary of an ncu report of one whole apply (every stage
kernel), using ncu_summary.py's metric set -- for profiles/.

    python tools/ncu_stages.py prof.ncu-rep out.json [label]
"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import KEYS, SCALE  # noqa: E402

rep, out = sys.argv[1], sys.argv[2]
label = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
res = []
for r in data:
    d = {"kernel": r[idx["Kernel Name"]][:90]}
    for k, name in KEYS.items():
        if k not in idx:
            continue
        try:
            v = float(r[idx[k]].replace(",", ""))
        except ValueError:
            continue
        d[name] = v * SCALE.get(units[idx[k]], 1.0)
    if d.get("fp64_tensor_ops") and d.get("duration"):
        d["tflops_under_ncu"] = d["fp64_tensor_ops"] / d["duration"] / 1e12
    if d.get("duration"):
        d["dram_gbs_under_ncu"] = (d.get("dram_read", 0) + d.get("dram_write", 0)) / d["duration"] / 1e9
    res.append(d)
json.dump({"label": label, "report": os.path.basename(rep), "launches": res}, open(out, "w"), indent=1)
print(out, len(res), "launches")
