"""Warp-stall samples of one kernel by SASS line, from an ncu report captured with
--set full --import-source on: totals inside / before / after the DMMA loop, the top
lines, and (with --dump A B) the lines A..B with their top stall reasons.

    python tools/ncu_source_stalls.py report.ncu-rep [--top 40] [--dump 600 700]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr, data = rows[hi], rows[hi + 1:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
num = lambda r, k: int(r[ix[k]] or 0)
tot = sum(num(r, "# Samples") for r in data)
dm = [i for i, r in enumerate(data) if "DMMA" in r[ix["Source"]]]
print(rows[0][1][:100] if len(rows[0]) > 1 else "", "| samples", tot, "| lines", len(data), "| DMMA lines", len(dm))


def region(a, b):
    agg = {k: 0 for k in stalls}
    s = 0
    for r in data[a:b]:
        s += num(r, "# Samples")
        for k in stalls:
            agg[k] += num(r, k)
    return s, [(k[6:], v) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:5]]


if dm:
    clusters, start, prev = [], dm[0], dm[0]
    for i in dm[1:]:
        if i - prev > 80:
            clusters.append((start, prev))
            start = i
        prev = i
    clusters.append((start, prev))
    for a, b in clusters:
        s, st = region(a, b + 1)
        print("DMMA loop lines %d-%d: %d samples (%.1f%%)" % (a, b, s, 100.0 * s / tot), st)
s, st = region(0, len(data))
print("all:", s, st)
for s, i in sorted(((num(r, "# Samples"), i) for i, r in enumerate(data)), reverse=True)[:top_n]:
    r = data[i]
    st = sorted(((num(r, k), k[6:]) for k in stalls), reverse=True)[:2]
    print("%6d  line %4d  x%-9s %-64s %s" % (s, i, r[ix["Instructions Executed"]], r[ix["Source"]][:64], st))
if "--dump" in sys.argv:
    a, b = int(sys.argv[sys.argv.index("--dump") + 1]), int(sys.argv[sys.argv.index("--dump") + 2])
    for i in range(a, b):
        r = data[i]
        s = num(r, "# Samples")
        st = sorted(((num(r, k), k[6:]) for k in stalls), reverse=True)[:2]
        print("%4d %6d x%-9s %-70s %s" % (i, s, r[ix["Instructions Executed"]], r[ix["Source"]][:70], st if s > 20 else ""))
