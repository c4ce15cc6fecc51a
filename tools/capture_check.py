"""User stream capture of qtt_apply (torch.cuda.graph): after a warm apply it
captures and replays correctly and later plain applies still work; as the
first use of a handle (no cached workspace yet) it is refused cleanly."""
import sys
import torch
import paper_1511_06029_b200 as q
import oracle
from qtt_workload import generate

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg, cores, x = generate(name)
xt = torch.from_numpy(x).cuda()
ref = oracle.apply_alg2(cores, x)
s = torch.cuda.Stream()
with q.QttOperator(cores) as op:
    op.apply(xt)
    torch.cuda.synchronize()
    y = torch.empty_like(xt)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        op.apply(xt, out=y)
    for _ in range(3):
        y.zero_()
        g.replay()
    torch.cuda.synchronize()
    oracle.assert_close(y.cpu().numpy(), ref)
    y2 = op.apply(xt)
    torch.cuda.synchronize()
    oracle.assert_close(y2.cpu().numpy(), ref)
    del g
print(name, "warm capture ok")
with q.QttOperator(cores) as op:
    g = torch.cuda.CUDAGraph()
    y = torch.empty_like(xt)
    try:
        with torch.cuda.graph(g, stream=s):
            op.apply(xt, out=y)
        print(name, "first-use capture unexpectedly accepted")
        sys.exit(1)
    except q.QttError as e:
        print(name, "first-use capture refused:", e)
    torch.cuda.synchronize()
    y3 = op.apply(xt)
    torch.cuda.synchronize()
    oracle.assert_close(y3.cpu().numpy(), ref)
print(name, "ok")
