"""Repeat split-K applies and compare bitwise with the first result (race hunt)."""
import sys
import numpy as np
import torch
import paper_1511_06029_b200 as q
from qtt_workload import generate, random_case
import oracle

def run(name, cores, x, reps=30):
    with q.QttOperator(cores) as op:
        print(name, [(s["k_first"], s["k_last"], s["variant"]) for s in op.stages()], op.stage_splits(x.shape[0]))
        xt = torch.from_numpy(x).cuda()
        ref = oracle.apply_alg2(cores, x)
        bad = 0
        y0 = op.apply(xt).cpu().numpy()
        try:
            oracle.assert_close(y0, ref)
        except AssertionError as e:
            print("  first result off:", str(e)[:200])
        for i in range(reps):
            y = op.apply(xt).cpu().numpy()
            if not np.array_equal(y, y0):
                bad += 1
                d = np.nonzero(y != y0)
                print("  rep", i, "differs at", len(d[-1]), "entries, first", d[-1][:8])
        print("  reps differing:", bad, "/", reps)

_, cores, x = generate("c3")
run("c3", cores, x)
for d, r, nrhs in ((12, 48, 1), (14, 32, 3), (16, 64, 1)):
    ranks = [1] + [r] * (d - 1) + [1]
    _, cores, x = random_case(9, d, r, nrhs, ranks=ranks)
    run(f"d{d} r{r}", cores, x)
