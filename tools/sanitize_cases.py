"""Small cases through every kernel variant, for compute-sanitizer (memcheck):
resident / merged / wide / generic stages, Morton tile + scalar kernels,
compressed matvec + densify, shard + projection, product, pipelined apply_host."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1511_06029_b200 as q  # noqa: E402
from paper_1511_06029_b200 import parallel as par  # noqa: E402
from qtt_workload import random_case, random_tt_vector  # noqa: E402

torch.cuda.set_device(0)
cases = [([1, 2, 5, 9, 16, 24, 48, 48, 33, 17, 8, 3, 1], 2, None),   # mixed stages
         ([1] + [20] * 9 + [1], 3, 1),                             # one level per launch
         ([1, 2, 70, 70, 5, 1], 1, 1),                             # wide single levels
         ([1, 2, 1501, 1501, 2, 1], 1, 1)]                          # generic kernel
for ranks, nrhs, maxL in cases:
    d = len(ranks) - 1
    _, cores, x = random_case(7, d, max(ranks), nrhs, ranks=ranks)
    with q.QttOperator(cores, max_stage_levels=maxL) as op:
        y = op.apply(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        print("apply", ranks[:4], [s["variant"] for s in op.stages()], float(y.abs().sum()))
# Morton: tiled (16-byte aligned) and scalar (8-byte aligned) kernels
g = torch.randn(1 << 15, dtype=torch.float64, device="cuda")
xq = q.morton_pack(g, 3, 5)
back = q.morton_unpack(xq, 3, 5)
base = torch.randn((1 << 12) + 1, dtype=torch.float64, device="cuda")
out = torch.empty_like(base)
q._lib.load().qtt_morton_pack(base[1:].data_ptr(), out[1:].data_ptr(), 2, 6, 1, None)
torch.cuda.synchronize()
print("morton", bool(torch.equal(back.view(-1), g)))
# compressed matvec + densify
_, A, _ = random_case(8, 11, 12, 1)
_, b = random_tt_vector(9, 11, 3)
with q.QttOperator(A) as op:
    c = op.compressed_matvec(b)
    cc = op.compressed_matvec(b, cores_only=True)
torch.cuda.synchronize()
print("compressed", float(c.abs().sum()), len(cc))
# shards (odd top rank padding) and a product
_, S, xs = random_case(10, 11, 33, 2)
for g_ in range(4):
    with par.QttShard(S, 2, g_) as sh:
        send = sh.apply(par.block_of(torch.from_numpy(xs).cuda(), g_, 4).contiguous())
torch.cuda.synchronize()
print("shard", float(send.abs().sum()))
_, M1, xm = random_case(11, 12, 6, 1)
_, M2, _ = random_case(12, 12, 9, 1)
with q.QttOperator(M1) as o1, q.QttOperator(M2) as o2, q.QttProduct([o1, o2]) as P:
    yp = P.apply(torch.from_numpy(xm).cuda())
torch.cuda.synchronize()
print("product", float(yp.abs().sum()))
# pipelined host apply (first / last stage in row chunks)
_, H, xh = random_case(13, 17, 10, 1)
with q.QttOperator(H) as op:
    yh = op.apply_host(xh)
print("apply_host", float(np.abs(yh).sum()))
print("ok")
