"""Race hunt on the BIE factors separately."""
import os
import sys
import numpy as np
import torch
import paper_1511_06029_b200 as q
from qtt_workload import bie_case

def hunt(name, f, xs, iters):
    refs = [f(v).clone() for v in xs]
    torch.cuda.synchronize()
    bad = []
    for i in range(iters):
        ys = [f(v) for v in xs]
        torch.cuda.synchronize()
        for j, (y, r) in enumerate(zip(ys, refs)):
            if not torch.equal(y, r):
                idx = torch.nonzero(y.view(-1) != r.view(-1)).view(-1)
                bad.append((i, j, int(idx.numel()), int(idx[0]), int(idx[-1])))
    print(name, os.environ.get("QTT_NO_PDL", ""), "mismatches", len(bad), bad[:4], flush=True)

rm, M, ry, Y, x = bie_case(0, 21, 9, 95, 50, 1)
x2 = np.ascontiguousarray(x[:, ::-1])
xs = [torch.from_numpy(v).cuda() for v in (x, x2)]
which = sys.argv[1] if len(sys.argv) > 1 else "MY"
with q.QttOperator(M) as opM, q.QttOperator(Y) as opY:
    if "Y" in which:
        print("Y stages", [(s["k_first"], s["k_last"], s["variant"], s["ksplit"]) for s in opY.stages()])
        hunt("Y", opY.apply, xs, 150)
    if "M" in which:
        print("M stages", [(s["k_first"], s["k_last"], s["variant"], s["ksplit"]) for s in opM.stages()])
        hunt("M", opM.apply, xs, 300)

if "P" in which:
    with q.QttOperator(M) as opM, q.QttOperator(Y) as opY, q.QttProduct([opM, opY]) as P:
        hunt("P", P.apply, xs, 200)
