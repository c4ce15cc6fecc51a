"""GPU parity for the Morton ordering kernels (NEXT-2; PAPER P:1625-1628,
Remark rem:interlace P:855-870; R18) and the grid apply.

A permutation is integer/index work: bitwise equality with the oracle's
permutation (oracle.morton, plain bit loops)."""
import numpy as np
import pytest

import oracle
from oracle import morton as OM
from qtt_workload import random_case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qtt():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    import paper_1511_06029_b200 as q
    q._lib.load()
    return q


@pytest.mark.parametrize("dim,levels,nrhs", [(1, 7, 2), (2, 3, 1), (2, 6, 2), (2, 7, 1), (3, 2, 3), (3, 3, 1),
                                             (3, 4, 2), (3, 5, 1), (3, 6, 1), (3, 5, 2), (2, 8, 3)])
def test_pack_unpack_bitwise(qtt, dim, levels, nrhs):
    N = 1 << (dim * levels)
    g = np.random.default_rng(dim * 100 + levels).standard_normal((nrhs, N))
    gt = torch.from_numpy(g).cuda()
    xq = qtt.morton_pack(gt, dim, levels)
    back = qtt.morton_unpack(xq, dim, levels)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(xq.cpu().numpy(), OM.pack(g, dim, levels))
    np.testing.assert_array_equal(back.cpu().numpy(), g)


def test_pack_full_size_sampled(qtt):
    """256^3 (the c4 grid, N = 2^24): sampled positions against the oracle's
    bit loops; round trip bitwise."""
    dim, levels = 3, 8
    N = 1 << 24
    g = torch.arange(N, dtype=torch.float64, device="cuda")     # value = natural index
    xq = qtt.morton_pack(g, dim, levels)
    back = qtt.morton_unpack(xq, dim, levels)
    torch.cuda.synchronize()
    assert torch.equal(back.view(-1), g)
    xh = xq.view(-1).cpu().numpy()
    rng = np.random.default_rng(7)
    for q in list(rng.integers(0, N, 2000)) + [0, 1, N - 1, N // 2, 4095, 4096]:
        c = OM.morton_coords(int(q), dim, levels)
        assert xh[q] == OM.natural_index(c, levels)


def test_morton_errors(qtt):
    lib = qtt._lib.load()
    a = torch.zeros(64, dtype=torch.float64, device="cuda")
    b = torch.zeros(64, dtype=torch.float64, device="cuda")
    E = qtt._lib
    assert lib.qtt_morton_pack(a.data_ptr(), b.data_ptr(), 4, 2, 1, None) == E.QTT_ERROR_INVALID_VALUE
    assert lib.qtt_morton_pack(a.data_ptr(), b.data_ptr(), 3, 0, 1, None) == E.QTT_ERROR_INVALID_VALUE
    assert lib.qtt_morton_pack(a.data_ptr(), a.data_ptr(), 3, 2, 1, None) == E.QTT_ERROR_INVALID_VALUE
    h = np.zeros(64)
    assert lib.qtt_morton_pack(h.ctypes.data, b.data_ptr(), 3, 2, 1, None) == E.QTT_ERROR_NOT_SUPPORTED
    with pytest.raises(ValueError):
        qtt.morton_pack(torch.zeros(63, dtype=torch.float64, device="cuda"), 3, 2)


@pytest.mark.parametrize("dim,levels,nrhs", [(3, 4, 2), (2, 6, 1), (3, 5, 1)])
def test_apply_grid(qtt, dim, levels, nrhs):
    d = dim * levels
    _, cores, _ = random_case(40 + d, d, 12, nrhs)
    g = np.random.default_rng(d).standard_normal((nrhs, 1 << d))
    op = qtt.QttOperator(cores)
    try:
        y = op.apply_grid(torch.from_numpy(g).cuda(), dim).cpu().numpy()
    finally:
        op.close()
    ref = OM.unpack(oracle.apply_alg2(cores, OM.pack(g, dim, levels)), dim, levels)
    oracle.assert_close(y, ref)


def test_pack_unaligned_pointers(qtt):
    """8-byte aligned (not 16) pointers take the per-element kernel: same result."""
    dim, levels = 3, 4
    N = 1 << 12
    base = torch.from_numpy(np.random.default_rng(2).standard_normal(N + 1)).cuda()
    g = base[1:]                                     # 8-byte offset view
    out = torch.empty(N + 1, dtype=torch.float64, device="cuda")[1:]
    lib = qtt._lib.load()
    assert lib.qtt_morton_pack(g.data_ptr(), out.data_ptr(), dim, levels, 1, None) == 0
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), OM.pack(g.cpu().numpy()[None, :], dim, levels)[0])


def test_morton_out_validation(qtt):
    """A caller's `out` of the wrong size is refused before the kernel runs."""
    g = torch.zeros((2, 1 << 12), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        qtt.morton_pack(g, 3, 4, out=torch.empty((1, 1 << 12), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        qtt.morton_unpack(g, 3, 4, out=torch.empty((3, 1 << 12), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        qtt.morton_pack(g, 3, 4, out=torch.empty((2, 1 << 12), dtype=torch.float32, device="cuda"))
