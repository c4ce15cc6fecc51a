"""Morton pack/unpack timing at 256^3: batched events, host wall per call, and a CUDA-graph replay."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1511_06029_b200 as q  # noqa: E402

N = 1 << 24
g = torch.randn(N, dtype=torch.float64, device="cuda")
x = torch.empty(1, N, dtype=torch.float64, device="cuda")
b = torch.empty_like(x)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for name, fn in (("pack", lambda: q.morton_pack(g, 3, 8, out=x, stream=s)),
                     ("unpack", lambda: q.morton_unpack(x, 3, 8, out=b, stream=s))):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        for _ in range(50):
            fn()
        e1.record(s)
        host = (time.perf_counter() - t0) / 50 * 1e3
        e1.synchronize()
        dev = e0.elapsed_time(e1) / 50
        print(f"{name}: batched {dev:.4f} ms/call ({16 * N / dev / 1e6:.0f} GB/s), host enqueue {host:.4f} ms/call")
