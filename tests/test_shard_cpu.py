"""Top-bit sharding, host side (-m "not gpu").

The shard plan's projection vectors come from the library's host-only
``qtt_shard_projection``; the local parts T_g (Alg. 2 levels 1..d-s on block g)
come from the oracle here (test infrastructure; on the GPU the shard kernels
compute them).  Checked: the decomposition y_h = sum_g T_g c_{h,g} equals the
oracle's full apply, in one process and across a world_size-2 gloo group
exchanging through ``parallel.exchange`` (the same call the NCCL path uses).
"""
import os
import socket

import numpy as np
import pytest

import oracle
from qtt_workload import random_case


@pytest.fixture(scope="module")
def par():
    from paper_1511_06029_b200 import build
    build.build()
    from paper_1511_06029_b200 import parallel
    return parallel


def local_part(cores, x_block, s):
    """Oracle T_g: Alg. 2 over the first d-s cores with the open bond r_{d-s}; (n, r)."""
    return oracle.alg2_sweep(cores[: len(cores) - s], x_block).T


@pytest.mark.parametrize("d,maxr,s", [(6, 3, 1), (8, 5, 2), (9, 7, 3), (10, 4, 1), (7, 6, 6)])
def test_decomposition_single_process(par, d, maxr, s):
    ranks, cores, x = random_case(1200 + d + s, d, maxr, 1)
    P = 1 << s
    if s >= d:
        pytest.skip("needs s < d")
    total = np.zeros((P, (1 << d) // P))
    for g in range(P):
        T = local_part(cores, par.block_of(x[0], g, P), s)
        W = par.shard_projection(cores, s, g)                 # (P, r_{d-s})
        total += W @ T.T                                       # send buffer [h][m]
    ref = oracle.apply_alg2(cores, x)[0]
    oracle.assert_close(total.reshape(1, -1), ref[None, :])


def test_projection_is_top_core_product(par):
    """c_{h,g}[a] is the QTT definition on the top s digits: for
    s = d - 1 ... check against oracle.entry on a rank-1 bottom core."""
    d, s = 4, 3
    ranks = [1, 3, 2, 4, 1]
    rng = np.random.default_rng(0)
    cores = [rng.standard_normal((ranks[k], 2, 2, ranks[k + 1])) for k in range(d)]
    e = np.zeros((1, 2, 2, ranks[1]))        # bottom core selecting bond alpha_1 = a when i_1 = j_1 = 0
    for g in range(1 << s):
        W = par.shard_projection(cores, s, g)
        for a in range(ranks[1]):
            e[:] = 0
            e[0, 0, 0, a] = 1.0
            for h in range(1 << s):
                # A'(i, j) with i = 2h, j = 2g: product of the top cores with alpha_1 = a
                ref = oracle.entry([e] + cores[1:], 2 * h, 2 * g)
                assert abs(W[h, a] - ref) <= 1e-14 * max(1.0, abs(ref))


def test_projection_validation(par):
    from paper_1511_06029_b200 import QttError
    _, cores, _ = random_case(5, 5, 3, 1)
    with pytest.raises(QttError):
        par.shard_projection(cores, 5, 0)       # s must be < d
    with pytest.raises(QttError):
        par.shard_projection(cores, 2, 4)       # part out of range


def _worker(rank, world, port, d, maxr, s, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from paper_1511_06029_b200 import parallel as par
        _, cores, x = random_case(1300 + d, d, maxr, 2)
        P = world
        blocks = [par.block_of(x, g, P) for g in range(P)]
        send = np.stack([par.shard_projection(cores, s, rank) @ local_part(cores, blocks[rank][r], s).T
                         for r in range(x.shape[0])])                 # [nrhs][P][n]
        out = torch.empty((x.shape[0], x.shape[1] // P), dtype=torch.float64)
        par.exchange(torch.from_numpy(send), out)
        ref = par.block_of(oracle.apply_alg2(cores, x), rank, P)
        err = float(np.abs(out.numpy() - ref).max() / np.abs(ref).max())
        q.put((rank, err))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("d,maxr", [(8, 4), (11, 9)])
def test_gloo_world2_exchange(par, d, maxr):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, d, maxr, 1, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(2))
    assert set(res) == {0, 1}
    assert max(res.values()) <= 1e-13, res
