"""Per-stage times of the BIE-shaped factors (qtt_workload.bie_case) at N = 2^21."""
import torch
import paper_1511_06029_b200 as q
from qtt_workload import bie_case

rm, M, ry, Y, x = bie_case(0, 21, 9, 95, 50, 1)
xt = torch.from_numpy(x).cuda()
for name, cores, ranks in (("M", M, rm), ("Y", Y, ry)):
    with q.QttOperator(cores) as op:
        y = op.apply(xt)
        torch.cuda.synchronize()
        op.set_stage_timing(True)
        op.stage_times()
        for _ in range(5):
            op.apply(xt, out=y)
        torch.cuda.synchronize()
        ms, n = op.stage_times()
        N = 1 << 21
        for s, t in zip(op.stages(), ms):
            k0, k1 = s["k_first"], s["k_last"]
            gb = 8 * N * (ranks[k0 - 1] + ranks[k1]) / (t / n * 1e-3) / 1e9
            print(name, k0, k1, s["variant"], s["ksplit"], "%.3f ms" % (t / n), "%.0f GB/s" % gb)
