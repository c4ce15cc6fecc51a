"""Per-stage times of c3 (and c4 given 'c4') applies: for A/B of wide-kernel switches
(e.g. QTT_WIDE_STAGGER_NS)."""
import sys

import torch

import paper_1511_06029_b200 as q
from qtt_workload import generate

for name in sys.argv[1:] or ["c3"]:
    cfg, cores, x = generate(name)
    with q.QttOperator(cores) as op:
        xt = torch.from_numpy(x).cuda()
        y = torch.empty_like(xt)
        for _ in range(3):
            op.apply(xt, out=y)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            op.apply(xt, out=y)
        b.record()
        b.synchronize()
        op.set_stage_timing(True)
        op.stage_times()
        for _ in range(5):
            op.apply(xt, out=y)
        torch.cuda.synchronize()
        ms, n = op.stage_times()
        st = op.stages()
        op.set_stage_timing(False)
        print(name, "ms/apply %.4f" % (a.elapsed_time(b) / 10),
              " ".join("%d-%d:%s %.4f" % (s_["k_first"], s_["k_last"], s_["variant"], ms[i] / n) for i, s_ in enumerate(st)))
