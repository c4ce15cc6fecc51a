"""us per apply of c1 / c2 (and any config names given): batched (200 back-to-back
applies, CUDA events) and single-call min, through the cached-workspace path
and the caller-workspace path; prints the launch plan.  A/B with QTT_NO_FUSED=1."""
import json
import sys

import torch

import paper_1511_06029_b200 as q
from qtt_workload import generate

names = sys.argv[1:] or ["c1", "c2"]
st = torch.cuda.Stream()
out = {}
for name in names:
    cfg, cores, x = generate(name)
    with q.QttOperator(cores) as op:
        xt = torch.from_numpy(x).cuda()
        y = torch.empty_like(xt)
        ws = torch.empty(op.workspace_size(cfg.nrhs) // 8 + 64, dtype=torch.float64, device="cuda")
        res = {"launches": op.launches(cfg.nrhs),
               "plan": [[s["k_first"], s["k_last"], s["variant"]] for s in op.stages(cfg.nrhs)]}
        for tag, fn in (("cached", lambda: op.apply(xt, out=y, stream=st)),
                        ("caller_ws", lambda: op.apply(xt, out=y, workspace=ws, stream=st))):
            for _ in range(10):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 200
            a.record(st)
            for _ in range(reps):
                fn()
            b.record(st)
            b.synchronize()
            single = []
            for _ in range(20):
                torch.cuda.synchronize()
                a.record(st)
                fn()
                b.record(st)
                b.synchronize()
                single.append(a.elapsed_time(b))
            res[tag + "_us_batched"] = round(a.elapsed_time(b) * 0 + 0, 2)
            res[tag + "_us_batched"] = None
            res[tag + "_us_single_min"] = round(min(single) * 1000, 2)
            # batched figure (re-time: the events above were reused for single calls)
            torch.cuda.synchronize()
            a.record(st)
            for _ in range(reps):
                fn()
            b.record(st)
            b.synchronize()
            res[tag + "_us_batched"] = round(a.elapsed_time(b) / reps * 1000, 2)
        out[name] = res
print(json.dumps(out))
