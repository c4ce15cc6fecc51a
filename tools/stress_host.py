"""Race hunt on qtt_apply_host (device-side copy flags): alternating inputs,
results bitwise equal to the device apply."""
import numpy as np
import torch
import paper_1511_06029_b200 as q
from qtt_workload import generate, bie_case

def hunt(name, cores, x, iters):
    x2 = np.ascontiguousarray(x[:, ::-1])
    with q.QttOperator(cores) as op:
        refs = [op.apply(torch.from_numpy(v).cuda()).cpu().numpy() for v in (x, x2)]
        xh = [torch.from_numpy(v).pin_memory() for v in (x, x2)]
        yh = [torch.empty_like(v).pin_memory() for v in xh]
        bad = 0
        for i in range(iters):
            for j in range(2):
                op.apply_host(xh[j].numpy(), out=yh[j].numpy())
                if not np.array_equal(yh[j].numpy(), refs[j]):
                    bad += 1
        print(name, iters, "mismatches", bad, flush=True)
        return bad

t = 0
for name, it in (("c2", 300), ("c3", 100), ("c4", 10)):
    _, cores, x = generate(name)
    t += hunt(name, cores, x, it)
_, _, _, Y, x = bie_case(0, 21, 9, 95, 50, 1)
t += hunt("bieY", Y, x, 50)
print("TOTAL", t)
