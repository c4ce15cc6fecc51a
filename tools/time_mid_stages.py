"""Per-stage times of constant-rank mid-size applies (d = 16..18): stage (levels, variant), ms, and the
stage's Alg. 2 / executed flop floor at the measured FP64 peak -- where the per-stage plan loses time
between the fused regime (d <= 15) and the DMMA-bound one (d >= 20).

    python tools/time_mid_stages.py [rank]
"""
import sys

import torch

import paper_1511_06029_b200 as q
from qtt_workload import random_case

r = int(sys.argv[1]) if len(sys.argv) > 1 else 16
for d in (16, 17, 18, 19):
    ranks = [1] + [min(r, 2 ** k, 2 ** (d - k)) for k in range(1, d)] + [1]
    _, cores, x = random_case(4242, d, r, 1, ranks=ranks)
    with q.QttOperator(cores) as op:
        xt = torch.from_numpy(x).cuda()
        y = torch.empty_like(xt)
        for _ in range(10):
            op.apply(xt, out=y)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(100):
            op.apply(xt, out=y)
        b.record()
        b.synchronize()
        op.set_stage_timing(True)
        op.stage_times()
        for _ in range(20):
            op.apply(xt, out=y)
        torch.cuda.synchronize()
        ms, n = op.stage_times()
        st = op.stages()
        op.set_stage_timing(False)
        N = 1 << d
        out = []
        for i, s_ in enumerate(st):
            k0, k1 = s_["k_first"], s_["k_last"]
            L = k1 - k0 + 1
            fl = 2.0 * N * (2 ** L) * ranks[k0 - 1] * ranks[k1]      # executed flops of the super-core GEMM
            out.append("%d-%d:%s %.1fus (floor %.1f)" % (k0, k1, s_["variant"], 1e3 * ms[i] / n, fl / 37.08e12 * 1e6))
        print("d", d, "r", r, "us/apply %.1f |" % (a.elapsed_time(b) * 10), " ".join(out))
