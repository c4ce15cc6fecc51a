"""Where the time of the compressed matvec (NEXT-3) goes: wall vs device time,
cores only vs dense, on the bench's c4 x rank-4 case."""
import statistics
import time

import torch

import paper_1511_06029_b200 as q
from qtt_workload import generate, random_tt_vector

dev = torch.device("cuda:0")
st = torch.cuda.Stream()
_, cA, _ = generate("c4", with_x=False)
_, bv = random_tt_vector(11, 24, 4)
with q.QttOperator(cA) as A:
    c = torch.empty(1 << 24, dtype=torch.float64, device=dev)
    import os
    once = os.environ.get("ONCE")
    for mode in (("dense",) if once else ("dense", "cores")):
        fn = (lambda: A.compressed_matvec(bv, out=c, stream=st)) if mode == "dense" else \
             (lambda: A.compressed_matvec(bv, stream=st, cores_only=True))
        fn()
        walls, devs = [], []
        for _ in range(1 if once else 7):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            a.record(st)
            fn()
            b.record(st)
            b.synchronize()
            walls.append((time.perf_counter() - t0) * 1e3)
            devs.append(a.elapsed_time(b))
        print(mode, "wall ms %.3f" % statistics.median(walls), "device ms %.3f" % statistics.median(devs))
