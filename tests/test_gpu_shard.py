"""GPU parity for top-bit sharding (NEXT-4), emulated on one GPU:
every part's shard plan runs on the same device one after another (no kernel
waits on another), the send buffers are summed, and block h must equal block
h of the full apply.  The ReduceScatter itself is covered on CPU with gloo
(tests/test_shard_cpu.py)."""
import numpy as np
import pytest

import oracle
from qtt_workload import generate, random_case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def par():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    from paper_1511_06029_b200 import parallel
    return parallel


def sharded_emulation(par, cores, x, s):
    P = 1 << s
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    total = None
    stages = None
    for g in range(P):
        with par.QttShard(cores, s, g) as sh:
            xb = par.block_of(xt, g, P).contiguous()
            send = sh.apply(xb)
            stages = sh.stages()
            total = send.clone() if total is None else total + send
    torch.cuda.synchronize()
    return total.reshape(x.shape[0], -1).cpu().numpy(), stages     # [nrhs][P*n] = y


@pytest.mark.parametrize("d,maxr,s,nrhs", [(8, 5, 1, 1), (10, 12, 2, 3), (12, 24, 3, 1), (13, 48, 1, 2),
                                           (11, 33, 2, 1), (9, 7, 5, 2), (14, 64, 3, 1)])
def test_sharded_equals_full(par, d, maxr, s, nrhs):
    _, cores, x = random_case(1400 + d + s, d, maxr, nrhs)
    y, stages = sharded_emulation(par, cores, x, s)
    assert stages[-1]["k_first"] == d - s + 1 and stages[-1]["k_last"] == d
    oracle.assert_close(y, oracle.apply_alg2(cores, x))


@pytest.mark.parametrize("s", [1, 2])
def test_sharded_block_diagonal_operator(par, s):
    """Shards of a BIE-shaped block-diagonal factor (qtt_workload.bie_case M):
    the local levels end in a diagonal stage, then the projection."""
    from qtt_workload import bie_case
    _, M, _, _, x = bie_case(6, 15, 6, 12, 8, 2)
    y, stages = sharded_emulation(par, M, x, s)
    assert any(st["variant"] == "diag" for st in stages), stages
    oracle.assert_close(y, oracle.apply_alg2(M, x))


def test_sharded_c3_p8(par):
    cfg, cores, x = generate("c3")
    y, _ = sharded_emulation(par, cores, x, 3)
    oracle.assert_close(y, oracle.apply_alg2(cores, x))


def test_shard_errors(par):
    _, cores, _ = random_case(1500, 8, 4, 1)
    import paper_1511_06029_b200 as q
    with pytest.raises(q.QttError):
        par.QttShard(cores, 8, 0)              # s must be < d
    with pytest.raises(q.QttError):
        par.QttShard(cores, 2, 4)              # part out of range
    with par.QttShard(cores, 1, 0) as sh:
        lib = q._lib.load()
        xb = torch.zeros(128, dtype=torch.float64, device="cuda")
        y = torch.zeros(256, dtype=torch.float64, device="cuda")
        # qtt_apply on a shard handle is rejected
        assert lib.qtt_apply(sh._h, xb.data_ptr(), y.data_ptr(), 1, None) == q._lib.QTT_ERROR_INVALID_VALUE
        with pytest.raises(ValueError):
            sh.apply(torch.zeros(64, dtype=torch.float64, device="cuda"))


# ------------------------------------------------------------------ fused exchange
@pytest.mark.parametrize("d,maxr,s,nrhs", [(10, 12, 1, 1), (12, 24, 2, 2), (13, 33, 3, 1), (11, 48, 2, 3)])
def test_fused_exchange_emulated(par, d, maxr, s, nrhs):
    """The projection stores every output block straight into its part's receive
    slot (the fused compute + exchange); here all P parts' buffers live on this
    one GPU and the parts run one after another (no kernel waits on another)."""
    _, cores, x = random_case(1600 + d + s, d, maxr, nrhs)
    P = 1 << s
    n = (1 << d) // P
    recv = [torch.empty((P, nrhs, n), dtype=torch.float64, device="cuda") for _ in range(P)]
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    for g in range(P):
        with par.QttShard(cores, s, g) as sh:
            sh.set_peers([r.data_ptr() for r in recv])
            sh.apply_fused(par.block_of(xt, g, P).contiguous())
    torch.cuda.synchronize()
    y = torch.empty((nrhs, 1 << d), dtype=torch.float64, device="cuda")
    for h in range(P):
        yh = torch.empty((nrhs, n), dtype=torch.float64, device="cuda")
        par.QttShard.reduce(recv[h], yh)
        y[:, h * n:(h + 1) * n] = yh
    torch.cuda.synchronize()
    oracle.assert_close(y.cpu().numpy(), oracle.apply_alg2(cores, x))


def _fused_worker(rank, world, port, q):
    import os
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1511_06029_b200 import parallel as par
        _, cores, x = random_case(1700, 12, 20, 2)
        x2 = np.ascontiguousarray(x[:, ::-1])
        op = par.ShardedQttOperator(cores, fused=True, max_nrhs=2)
        refs = [par.block_of(oracle.apply_alg2(cores, v), rank, world) for v in (x, x2)]
        xbs = [par.block_of(torch.from_numpy(np.ascontiguousarray(v)).cuda(), rank, world).contiguous()
               for v in (x, x2)]
        errs = []
        # stream-ordered applies back to back (no host sync between them), alternating inputs
        ys = [op.apply(xbs[i % 2]) for i in range(6)]
        ys.append(op.apply(xbs[0][:1].contiguous()))          # nrhs 1 < max_nrhs
        for i, y in enumerate(ys[:6]):
            ref = refs[i % 2]
            errs.append(float(np.abs(y.cpu().numpy() - ref).max() / np.abs(ref).max()))
        errs.append(float(np.abs(ys[6].cpu().numpy() - refs[0][:1]).max() / np.abs(refs[0][:1]).max()))
        op.close()
        q.put((rank, max(errs)))
    finally:
        dist.destroy_process_group()


def test_fused_exchange_two_processes_ipc(par):
    """Two processes on this one GPU: receive buffers shared through CUDA IPC,
    cross-process ordering by interprocess CUDA events (stream waits) behind
    host-only gloo barriers -- no device synchronisation, and no kernel waits on
    another process's kernel."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fused_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(2))
    assert max(res.values()) <= 1e-12, res
