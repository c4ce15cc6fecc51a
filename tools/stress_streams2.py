"""Race hunt: where do wrong c3 outputs sit (last stage tile / warp / lane)?"""
import collections
import numpy as np
import torch
import paper_1511_06029_b200 as q
from qtt_workload import generate

cfg, cores, x = generate("c3")
x2 = np.ascontiguousarray(x[:, ::-1])
N = 1 << 21
Q = N // 128
with q.QttOperator(cores) as op:
    ref1 = op.apply(torch.from_numpy(x).cuda()).clone()
    ref2 = op.apply(torch.from_numpy(x2).cuda()).clone()
    torch.cuda.synchronize()
    xa, xb = torch.from_numpy(x).cuda(), torch.from_numpy(x2).cuda()
    for i in range(60):
        y = op.apply(xa if i % 2 == 0 else xb)
        torch.cuda.synchronize()
        ref = ref1 if i % 2 == 0 else ref2
        if not torch.equal(y, ref):
            p = torch.nonzero(y.view(-1) != ref.view(-1)).view(-1).cpu().numpy()
            m, ii = p % Q, p // Q
            rt, rg, cg = m // 64, (m % 64) // 16, ii // 32
            lane = (m % 8) * 4 + (ii % 8) // 2
            keys = collections.Counter(zip(rt.tolist(), rg.tolist(), cg.tolist()))
            yo = y.view(-1)[torch.from_numpy(p).cuda()].cpu().numpy()
            ro = ref.view(-1)[torch.from_numpy(p).cuda()].cpu().numpy()
            other = (ref2 if i % 2 == 0 else ref1).view(-1)[torch.from_numpy(p).cuda()].cpu().numpy()
            print(f"iter {i}: {len(p)} wrong; (tile,rg,cg) groups {dict(keys)}; lanes {sorted(set(lane.tolist()))[:40]}")
            print("   rel err", float(np.max(np.abs(yo - ro) / (np.abs(ro) + 1e-300))), "close to other-input result:",
                  float(np.max(np.abs(yo - other) / (np.abs(other) + 1e-300))))
