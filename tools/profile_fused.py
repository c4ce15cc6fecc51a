"""Run a few applies of the given configs (default c1 c2) -- a driver for
QTT_FUSED_PROFILE=1 (in-kernel stage/barrier timestamps) and for ncu."""
import sys

import torch

import paper_1511_06029_b200 as q
from qtt_workload import generate

grid = "--grid" in sys.argv
names = [a for a in sys.argv[1:] if not a.startswith("--")]
for name in names or ["c1", "c2"]:
    cfg, cores, x = generate(name)
    with q.QttOperator(cores) as op:
        xt = torch.from_numpy(x).cuda()
        y = torch.empty_like(xt)
        for _ in range(5):
            if grid:
                op.apply_grid(xt, 3, out=y)
            else:
                op.apply(xt, out=y)
        torch.cuda.synchronize()
        print(name, "plan", [[s["k_first"], s["k_last"], s["variant"]] for s in op.stages(cfg.nrhs)], flush=True)
