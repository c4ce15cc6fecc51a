"""ms per apply (batched, CUDA events) of the BASELINE configs; A/B helper."""
import sys
import torch
import paper_1511_06029_b200 as q
from qtt_workload import generate

names = sys.argv[1:] or ["c1", "c2", "c3", "c4"]
st = torch.cuda.Stream()
out = {}
for name in names:
    cfg, cores, x = generate(name)
    with q.QttOperator(cores) as op:
        xt = torch.from_numpy(x).cuda()
        y = torch.empty_like(xt)
        ws = torch.empty(op.workspace_size(cfg.nrhs) // 8 + 64, dtype=torch.float64, device="cuda")
        reps = 5 if name in ("c4", "c5") else 50
        fn = lambda: op.apply(xt, out=y, workspace=ws, stream=st)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        b.synchronize()
        out[name] = round(a.elapsed_time(b) / reps * 1000, 2)
print("us/apply", out)
