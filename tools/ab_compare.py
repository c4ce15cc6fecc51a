"""Compare two bench JSON lines stage by stage: python tools/ab_compare.py A.json B.json"""
import json
import sys

a, b = (json.load(open(p)) for p in sys.argv[1:3])
print("c4 ms/apply: A %.3f  B %.3f" % (a["ms_per_step"], b["ms_per_step"]))
for sa, sb in zip(a["per_stage_roofline"]["stages"], b["per_stage_roofline"]["stages"]):
    print("  c4", sa["levels"], sa["variant"], "%.3f -> %.3f ms" % (sa["ms"], sb["ms"]))
ea, eb = a["other_configs_and_next_rows"], b["other_configs_and_next_rows"]
for k in ea:
    va, vb = ea[k], eb.get(k, {})
    ms_a = va.get("ms_per_apply", va.get("pack_ms", va.get("ms_wall_median")))
    ms_b = vb.get("ms_per_apply", vb.get("pack_ms", vb.get("ms_wall_median")))
    print(k, "A %.4f  B %.4f ms" % (ms_a, ms_b))
    if "stages" in va and len(va["stages"][0]) > 3:
        for x, y in zip(va["stages"], vb["stages"]):
            print("    ", x[:3], "%.4f -> %.4f" % (x[3], y[3]))
