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
