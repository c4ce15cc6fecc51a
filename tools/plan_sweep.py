import torch, paper_1511_06029_b200 as q
from qtt_workload import generate
st = torch.cuda.Stream()
def t(op, x, reps=300):
    y = torch.empty_like(x)
    for _ in range(10): op.apply(x, out=y, stream=st)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): op.apply(x, out=y, stream=st)
    b.record(st); b.synchronize()
    return a.elapsed_time(b) / reps * 1000
for name in ("c1", "c2"):
    cfg, cores, x = generate(name)
    xt = torch.from_numpy(x).cuda()
    for L in (2, 3, 4, 5, 6, 8, 10):
        with q.QttOperator(cores, max_stage_levels=L) as op:
            print(name, L, [(s["k_first"], s["k_last"], s["variant"][0]) for s in op.stages()], "%.2f us" % t(op, xt))
