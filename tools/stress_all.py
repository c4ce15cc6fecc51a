"""Long race hunt: many back-to-back applies with alternating inputs (no host
sync between the two of a pair), every result bitwise equal to its reference."""
import sys
import numpy as np
import torch
import paper_1511_06029_b200 as q
from qtt_workload import generate, bie_case

def hunt(name, op_apply, xs, iters):
    refs = [op_apply(v).clone() for v in xs]
    torch.cuda.synchronize()
    bad = 0
    for i in range(iters):
        ys = [op_apply(v) for v in xs]           # both enqueued before any sync
        torch.cuda.synchronize()
        for y, r in zip(ys, refs):
            if not torch.equal(y, r):
                bad += 1
    print(name, "iterations", iters, "mismatches", bad, flush=True)
    return bad

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
total = 0
for name, iters in (("c3", 150), ("c2", 400), ("c1", 400), ("c4", 20)):
    iters = int(iters * scale)
    cfg, cores, x = generate(name)
    x2 = np.ascontiguousarray(x[:, ::-1])
    with q.QttOperator(cores) as op:
        total += hunt(name, op.apply, [torch.from_numpy(v).cuda() for v in (x, x2)], iters)
rm, M, ry, Y, x = bie_case(0, 21, 9, 95, 50, 1)
x2 = np.ascontiguousarray(x[:, ::-1])
with q.QttOperator(M) as opM, q.QttOperator(Y) as opY, q.QttProduct([opM, opY]) as P:
    total += hunt("bie", P.apply, [torch.from_numpy(v).cuda() for v in (x, x2)], int(60 * scale))
print("TOTAL", total)
sys.exit(1 if total else 0)
