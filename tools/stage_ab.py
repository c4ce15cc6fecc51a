import torch, paper_1511_06029_b200 as q
from qtt_workload import generate
for name in ("c4", "c5"):
    cfg, cores, x = generate(name)
    with q.QttOperator(cores) as op:
        xt = torch.from_numpy(x).cuda(); y = torch.empty_like(xt)
        op.apply(xt, out=y); torch.cuda.synchronize()
        op.set_stage_timing(True); op.stage_times()
        for _ in range(3): op.apply(xt, out=y)
        torch.cuda.synchronize()
        ms, n = op.stage_times()
        st = op.stages()
        print(name, "first", st[0]["k_first"], st[0]["k_last"], "%.3f" % (ms[0]/n), "last", st[-1]["k_first"], st[-1]["k_last"], "%.3f" % (ms[-1]/n), "total %.2f" % (sum(ms)/n))
