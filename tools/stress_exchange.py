"""Race hunt on the fused shard exchange: two processes sharing this GPU,
CUDA IPC receive buffers + interprocess events, 100 back-to-back applies with
alternating inputs; every block compared with the oracle-free reference
(the single-process QttOperator apply of the full vector)."""
import os
import socket
import sys

import numpy as np
import torch
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port, q, iters):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    import paper_1511_06029_b200 as qq
    from paper_1511_06029_b200 import parallel as par
    from qtt_workload import random_case
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, cores, x = random_case(1800, 16, 24, 1)
    x2 = np.ascontiguousarray(x[:, ::-1])
    with qq.QttOperator(cores) as full:
        refs = [par.block_of(full.apply(torch.from_numpy(v).cuda()), rank, world).clone() for v in (x, x2)]
    op = par.ShardedQttOperator(cores, fused=True, max_nrhs=1)
    xb = [par.block_of(torch.from_numpy(v).cuda(), rank, world).contiguous() for v in (x, x2)]
    worst = 0.0
    for i in range(iters):
        ys = [op.apply(xb[j]) for j in range(2)]
        for j in range(2):
            err = float((ys[j] - refs[j]).abs().max() / refs[j].abs().max())
            worst = max(worst, err)
    op.close()
    q.put((rank, worst))
    dist.destroy_process_group()


if __name__ == "__main__":
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q, 100)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    res = dict(q.get(timeout=10) for _ in range(2))
    print("worst relative error per rank", res)
    sys.exit(0 if max(res.values()) < 1e-12 else 1)
