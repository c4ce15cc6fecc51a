"""Applies with N * nrhs > 2^31 (reading: launch groups).

Every launch keeps N * group <= 2^31 rows (32-bit TMA row coordinates); an
apply with more right-hand sides runs as consecutive RHS groups, and
qtt_apply also lowers the group while its workspace would not fit in free
device memory.  The RHS are independent problems, so each column must be
bitwise what a one-RHS apply gives.  Expected values: the exact cyclic shift
(torch.roll, a library routine) and exact power-of-two scalings of the
pinned c5 result.
"""
import numpy as np
import pytest

import oracle
from qtt_workload import closed_forms as CF
from qtt_workload import generate

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qtt():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    import paper_1511_06029_b200 as q
    q._lib.load()
    return q


def _free_gb():
    torch.cuda.empty_cache()
    return torch.cuda.mem_get_info()[0] / 2**30


def test_shift_d30_nrhs4_beyond_2_31(qtt):
    """d = 30, 4 RHS: 2^32 rows in all, two launch groups of 2^31."""
    d, nrhs, s = 30, 4, 123457
    N = 1 << d
    if _free_gb() < 140:
        pytest.skip("needs ~130 GB of free device memory")
    x = torch.arange(N * nrhs, dtype=torch.float64, device="cuda").view(nrhs, N)   # exact integers
    y = torch.empty_like(x)
    op = qtt.QttOperator(CF.shift_cores(d, s))
    try:
        assert op.workspace_size(nrhs) == op.workspace_size(2)      # sized for one group of 2
        op.apply(x, out=y)
        torch.cuda.synchronize()
        assert torch.equal(y, torch.roll(x, s, dims=1))
    finally:
        op.close()
    del y
    torch.cuda.empty_cache()
    # the caller-workspace entry point groups the same way
    op = qtt.QttOperator(CF.shift_cores(d, -s))
    try:
        ws = torch.empty(op.workspace_size(nrhs) // 8 + 64, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        op.apply(x, out=y, workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(y, torch.roll(x, -s, dims=1))
    finally:
        op.close()


def test_c5_many_rhs_memory_groups(qtt):
    """c5 with 17 RHS: the workspace of one launch for all 17 (~0.9 TB) exceeds
    HBM, so qtt_apply runs memory-bounded RHS groups.  x_s = +-2^(s mod 4) x:
    scaling by powers of two is exact, so y_s = +-2^(s mod 4) y bitwise."""
    cfg, cores, x = generate("c5")
    nrhs = 17
    if _free_gb() < 150:
        pytest.skip("needs ~140 GB of free device memory")
    op = qtt.QttOperator(cores)
    try:
        x1 = torch.from_numpy(x).cuda()
        y1 = op.apply(x1)
        torch.cuda.synchronize()
        scale = torch.tensor([(-1.0) ** s * 2.0 ** (s % 4) for s in range(nrhs)], dtype=torch.float64,
                             device="cuda").view(nrhs, 1)
        xs = x1 * scale
        del x1
        ys = op.apply(xs)
        torch.cuda.synchronize()
        assert torch.equal(ys, y1 * scale)
        # y1 itself: every entry against the chunked oracle in test_gpu_full_parity.py
    finally:
        op.close()
        torch.cuda.empty_cache()
