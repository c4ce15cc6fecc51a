"""Launch-latency floor: applies of tiny operators (identity = one diag stage)."""
import torch
import paper_1511_06029_b200 as q
from qtt_workload import closed_forms as CF, generate

st = torch.cuda.Stream()

def t(op, x, reps=200):
    y = torch.empty_like(x)
    for _ in range(5):
        op.apply(x, out=y, stream=st)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        op.apply(x, out=y, stream=st)
    b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / reps * 1000

for d in (12, 15):
    with q.QttOperator(CF.identity_cores(d)) as op:
        x = torch.randn(1, 1 << d, dtype=torch.float64, device="cuda")
        print("identity d=%d" % d, [s["variant"] for s in op.stages()], "%.2f us" % t(op, x))
    with q.QttOperator(CF.identity_cores(d), max_stage_levels=1) as op:
        print("identity d=%d one launch per level" % d, op.launches_per_apply, "%.2f us" % t(op, x))
for name in ("c1", "c2"):
    cfg, cores, x = generate(name)
    with q.QttOperator(cores) as op:
        xt = torch.from_numpy(x).cuda()
        print(name, [(s["k_first"], s["k_last"], s["variant"]) for s in op.stages()], "%.2f us" % t(op, xt))
