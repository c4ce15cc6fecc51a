"""Race hunt for the fused one-launch apply (grid barrier, counter reset across
launches, split barrier with the super-core prefetch) and the streaming
diagonal stage: thousands of back-to-back applies with alternating inputs,
through the cached workspace, a caller workspace (counter cleared by a stream
op), two streams, the grid apply and nrhs = 2; every result bitwise equal to
its reference.  Exit status 1 on any mismatch."""
import sys

import numpy as np
import torch

import paper_1511_06029_b200 as q
from qtt_workload import bie_case, generate

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
total = 0


def hunt(name, fns, iters):
    global total
    refs = []
    for f in fns:          # sync before the clone: some calls run on side streams
        y = f()
        torch.cuda.synchronize()
        refs.append(y.clone())
    bad = [0] * len(fns)
    for _ in range(iters):
        ys = [f() for f in fns]                  # all enqueued before any sync
        torch.cuda.synchronize()
        for i, (y, r) in enumerate(zip(ys, refs)):
            bad[i] += not torch.equal(y, r)
    print(name, "iterations", iters, "x", len(fns), "mismatches per call", bad, flush=True)
    bad = sum(bad)
    total += bad


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name in ("c1", "c2"):
    cfg, cores, x = generate(name)
    xs = [torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (x, x[:, ::-1], -x)]
    x2 = torch.cat([xs[0], xs[1]]).contiguous()
    with q.QttOperator(cores) as op:
        assert op.launches(1) == 1
        ws = torch.empty(op.workspace_size(2) // 8 + 64, dtype=torch.float64, device="cuda")
        fns = [lambda: op.apply(xs[0]),
               lambda: op.apply(xs[1], stream=s1),
               lambda: op.apply(xs[2], workspace=ws, stream=s2),
               lambda: op.apply(x2),
               lambda: op.apply_grid(xs[0], 3)]
        hunt(name + " fused", fns, int(400 * scale))
rm, M, ry, Y, x = bie_case(0, 21, 9, 95, 50, 1)
xs = [torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (x, x[:, ::-1])]
with q.QttOperator(M) as opM:
    hunt("bie M (diag stream)", [lambda: opM.apply(xs[0]), lambda: opM.apply(xs[1])], int(100 * scale))
print("TOTAL", total)
sys.exit(1 if total else 0)
