"""us per apply: plain apply vs grid apply (natural-order 3-D grid in and out)
for c1 / c2, fused (one launch) and per-stage (Morton pack + stages + unpack)."""
import json
import sys

import torch

import paper_1511_06029_b200 as q
from qtt_workload import generate


def t(fn, st, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    b.synchronize()
    return round(a.elapsed_time(b) / reps * 1e3, 2)


st = torch.cuda.Stream()
out = {}
for name in sys.argv[1:] or ["c1", "c2"]:
    cfg, cores, x = generate(name)
    xt = torch.from_numpy(x).cuda()
    y = torch.empty_like(xt)
    r = {}
    for fused in (True, False):
        with q.QttOperator(cores, fused=fused) as op:
            tag = "fused" if fused else "per_stage"
            r[tag + "_plain_us"] = t(lambda: op.apply(xt, out=y, stream=st), st)
            r[tag + "_grid_us"] = t(lambda: op.apply_grid(xt, 3, out=y, stream=st), st)
    out[name] = r
print(json.dumps(out))
