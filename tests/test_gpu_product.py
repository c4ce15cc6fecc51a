"""GPU parity for products of QTT operators (NEXT-1; the paper's BIE
preconditioner X = M Y applied as two QTT matvecs).

Expected values come from the oracle on the COMPOSED operator (oracle.compose,
the rank-product cores of P:1226-1231, pinned in test_oracle_pins.py), an
independent path from applying the factors one after another."""
import numpy as np
import pytest

import oracle
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


@pytest.mark.parametrize("d,rm,ry,nrhs", [(10, 4, 9, 1), (12, 6, 17, 3), (13, 3, 24, 2), (9, 1, 5, 1)])
def test_two_factor_product(qtt, d, rm, ry, nrhs):
    _, M, x = random_case(500 + d, d, rm, nrhs)
    _, Y, _ = random_case(600 + d, d, ry, nrhs)
    ref = oracle.apply_alg2(oracle.compose(M, Y), x)
    with qtt.QttOperator(M) as opM, qtt.QttOperator(Y) as opY, qtt.QttProduct([opM, opY]) as P:
        y = P.apply(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        oracle.assert_close(y.cpu().numpy(), ref)
        # same result as applying the factors one after another on the GPU (bitwise)
        y2 = opM.apply(opY.apply(torch.from_numpy(x).cuda()))
        torch.cuda.synchronize()
        assert torch.equal(y, y2)


def test_three_factors_caller_workspace(qtt):
    d, nrhs = 11, 2
    fs = [random_case(700 + i, d, 6 + 3 * i, nrhs)[1] for i in range(3)]
    x = np.random.default_rng(3).standard_normal((nrhs, 1 << d))
    ref = oracle.apply_alg2(oracle.compose(oracle.compose(fs[0], fs[1]), fs[2]), x)
    ops = [qtt.QttOperator(c) for c in fs]
    try:
        P = qtt.QttProduct(ops)
        ws = torch.empty(P.workspace_size(nrhs) // 8 + 64, dtype=torch.float64, device="cuda")
        y = P.apply(torch.from_numpy(x).cuda(), workspace=ws)
        torch.cuda.synchronize()
        oracle.assert_close(y.cpu().numpy(), ref)
        P.close()
    finally:
        for o in ops:
            o.close()


def test_single_factor_is_apply(qtt):
    _, A, x = random_case(800, 12, 20, 1)
    with qtt.QttOperator(A) as op, qtt.QttProduct([op]) as P:
        xt = torch.from_numpy(x).cuda()
        assert torch.equal(P.apply(xt), op.apply(xt))


def test_product_errors(qtt):
    _, A, _ = random_case(801, 10, 4, 1)
    _, B, _ = random_case(802, 11, 4, 1)
    with qtt.QttOperator(A) as a, qtt.QttOperator(B) as b:
        with pytest.raises(qtt.QttError):
            qtt.QttProduct([a, b])          # different d
    with pytest.raises(ValueError):
        qtt.QttProduct([])


@pytest.mark.parametrize("d,point_bits,nrhs", [(14, 9, 1), (16, 9, 2)])
def test_bie_shaped_product(qtt, d, point_bits, nrhs):
    """The boundary-integral preconditioner shape (qtt_workload.bie_case: Y with
    ranks up to 95, block-diagonal M with ranks up to 50, Table 3): the product
    against the oracle applying the factors in turn (the composed rank 4750
    would be too large for the oracle's dense algebra)."""
    from qtt_workload import bie_case
    _, M, _, Y, x = bie_case(7, d, point_bits, 95, 50, nrhs)
    ref = oracle.apply_alg2(M, oracle.apply_alg2(Y, x))
    with qtt.QttOperator(M) as opM, qtt.QttOperator(Y) as opY, qtt.QttProduct([opM, opY]) as P:
        y = P.apply(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
    oracle.assert_close(y.cpu().numpy(), ref)
