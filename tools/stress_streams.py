"""Race hunt: c3 applies back to back on two streams (shared cached workspace)."""
import numpy as np
import torch
import paper_1511_06029_b200 as q
from qtt_workload import generate

cfg, cores, x = generate("c3")
x2 = np.ascontiguousarray(x[:, ::-1])
bad = 0
with q.QttOperator(cores) as op:
    ref1 = op.apply(torch.from_numpy(x).cuda()).clone()
    ref2 = op.apply(torch.from_numpy(x2).cuda()).clone()
    torch.cuda.synchronize()
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    xa, xb = torch.from_numpy(x).cuda(), torch.from_numpy(x2).cuda()
    torch.cuda.synchronize()
    for i in range(40):
        ya = op.apply(xa, stream=a)
        yb = op.apply(xb, stream=b)
        a.synchronize()
        b.synchronize()
        ok = torch.equal(ya, ref1) and torch.equal(yb, ref2)
        if not ok:
            bad += 1
            print("iter", i, "a diff", int((ya != ref1).sum()), "b diff", int((yb != ref2).sum()))
    # same stream, many
    for i in range(40):
        y = op.apply(xa)
        torch.cuda.synchronize()
        if not torch.equal(y, ref1):
            bad += 1
            print("same-stream iter", i, "diff", int((y != ref1).sum()))
print("bad", bad)
