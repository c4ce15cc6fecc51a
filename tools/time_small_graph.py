"""c1 / c2 per-apply time three ways, to separate host enqueue cost from device time:
  host_us      -- wall time of one op.apply() call on the host (no sync; ctypes + validation + enqueue)
  stream_us    -- 200 back-to-back op.apply() calls, CUDA events (what bench.py's extras report)
  graph_us     -- 100 applies captured in ONE CUDA graph, replayed (no host work between applies)
With QTT_NO_FUSED=1 the per-stage plan is timed instead."""
import json
import sys
import time

import torch

import paper_1511_06029_b200 as q
from qtt_workload import generate

names = sys.argv[1:] or ["c1", "c2"]
st = torch.cuda.Stream()
out = {}
for name in names:
    cfg, cores, x = generate(name)
    with q.QttOperator(cores) as op:
        xt = torch.from_numpy(x).cuda()
        y = torch.empty_like(xt)
        res = {"plan": [[s["k_first"], s["k_last"], s["variant"]] for s in op.stages(cfg.nrhs)]}
        for _ in range(20):
            op.apply(xt, out=y, stream=st)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(300):
            op.apply(xt, out=y, stream=st)
        res["host_us"] = round((time.perf_counter() - t0) / 300 * 1e6, 2)
        # the C ABI alone (ctypes call with prepared arguments, no torch validation)
        lib = q._lib.load()
        hx, hy, hs = xt.data_ptr(), y.data_ptr(), st.cuda_stream
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(300):
            lib.qtt_apply(op.handle, hx, hy, cfg.nrhs, hs)
        res["host_c_us"] = round((time.perf_counter() - t0) / 300 * 1e6, 2)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(200):
            op.apply(xt, out=y, stream=st)
        b.record(st)
        b.synchronize()
        res["stream_us"] = round(a.elapsed_time(b) / 200 * 1000, 2)
        g = torch.cuda.CUDAGraph()
        reps = 100
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                op.apply(xt, out=y)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        best = []
        for _ in range(5):
            a.record(st)
            with torch.cuda.stream(st):
                g.replay()
            b.record(st)
            b.synchronize()
            best.append(a.elapsed_time(b) / reps * 1000)
        res["graph_us"] = round(min(best), 2)
        res["graph_us_median"] = round(sorted(best)[2], 2)
        ref = op.apply(xt).clone()
        torch.cuda.synchronize()
        res["graph_result_bitwise"] = bool(torch.equal(y, ref))
        del g
        out[name] = res
print(json.dumps(out))
