"""A/B of stage splits for one config: per-stage and whole-apply times of the
default plan and of each QTT_PLAN_FORCE_STAGES spec given (each in its own
process: the switch is read once).  Usage: python tools/ab_stages.py c4 "1-7,8-9,...,18-24" ..."""
import json
import os
import subprocess
import sys

CHILD = r"""
import json, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_1511_06029_b200 as q
from qtt_workload import generate
cfg, cores, x = generate(sys.argv[2])
with q.QttOperator(cores) as op:
    xt = torch.from_numpy(x).cuda(); y = torch.empty_like(xt)
    for _ in range(3): op.apply(xt, out=y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): op.apply(xt, out=y)
    b.record(); b.synchronize()
    total = a.elapsed_time(b) / 10
    op.set_stage_timing(True); op.stage_times()
    for _ in range(5): op.apply(xt, out=y)
    torch.cuda.synchronize()
    ms, n = op.stage_times()
    st = op.stages()
    op.set_stage_timing(False)
    print(json.dumps({"ms_per_apply": total, "stages": [[s["k_first"], s["k_last"], s["variant"], round(ms[i] / n, 4)]
                                                        for i, s in enumerate(st)]}))
"""

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
name = sys.argv[1]
out = {}
for spec in ["default"] + sys.argv[2:]:
    env = dict(os.environ)
    if spec != "default":
        env["QTT_PLAN_FORCE_STAGES"] = spec
    r = subprocess.run([sys.executable, "-c", CHILD, root, name], env=env, capture_output=True, text=True)
    out[spec] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
print(json.dumps(out, indent=1))
