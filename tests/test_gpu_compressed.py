"""GPU parity for the QTT-compressed matvec and TT-vector densification
(NEXT-3; PAPER section 4.2).

Expected values: oracle.compressed_matvec + oracle.tt_vector_dense (pinned in
test_oracle_pins.py), and independently oracle.apply_alg2 on the densified b."""
import numpy as np
import pytest

import oracle
from qtt_workload import generate, random_case, random_tt_vector

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qtt():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    import paper_1511_06029_b200 as q
    q._lib.load()
    return q


CASES = [  # d, max rank of A, max rank of b
    (1, 1, 1), (2, 2, 2), (3, 3, 2), (7, 5, 3), (10, 9, 4), (11, 16, 3), (13, 24, 5), (12, 48, 6), (15, 8, 2),
]


@pytest.mark.parametrize("d,ra,rb", CASES)
def test_compressed_dense(qtt, d, ra, rb):
    _, A, _ = random_case(900 + d, d, ra, 1)
    _, b = random_tt_vector(950 + d, d, rb)
    with qtt.QttOperator(A) as op:
        c = op.compressed_matvec(b).cpu().numpy()
    ref = oracle.tt_vector_dense(oracle.compressed_matvec(A, b))
    oracle.assert_close(c[None, :], ref[None, :])
    # independent path: the uncompressed apply of the densified b
    oracle.assert_close(c[None, :], oracle.apply_alg2(A, oracle.tt_vector_dense(b)[None, :]))


@pytest.mark.parametrize("d,ra,rb", [(6, 4, 3), (12, 20, 5)])
def test_compressed_cores(qtt, d, ra, rb):
    _, A, _ = random_case(910 + d, d, ra, 1)
    _, b = random_tt_vector(960 + d, d, rb)
    with qtt.QttOperator(A) as op:
        cores = [t.cpu().numpy() for t in op.compressed_matvec(b, cores_only=True)]
    ref = oracle.compressed_matvec(A, b)
    for C, R in zip(cores, ref):
        assert C.shape == R.shape
        np.testing.assert_allclose(C, R, rtol=1e-14, atol=1e-15 * np.abs(R).max())


def test_compressed_full_size_c4(qtt):
    """c4's operator (N = 2^24) times a rank-3 TT vector: sampled entries of the
    dense result against the oracle's TT entries of the product cores."""
    cfg, A, _ = generate("c4", with_x=False)
    _, b = random_tt_vector(77, cfg.d, 3)
    with qtt.QttOperator(A) as op:
        c = op.compressed_matvec(b).cpu().numpy()
    rows = np.unique(np.r_[np.random.default_rng(3).integers(0, cfg.N, 1500), [0, 1, cfg.N - 1]])
    ref = oracle.tt_vector_entries(oracle.compressed_matvec(A, b), rows)
    rms = float(np.sqrt(np.mean(ref ** 2)))
    oracle.assert_close(c[rows][None, :], ref[None, :], rms=rms)


def test_compressed_errors(qtt):
    _, A, _ = random_case(920, 6, 4, 1)
    _, b = random_tt_vector(921, 5, 2)
    with qtt.QttOperator(A) as op:
        with pytest.raises(ValueError):
            op.compressed_matvec(b)                  # wrong d
        _, b6 = random_tt_vector(922, 6, 2)
        b6[0] = np.zeros((2, 2, b6[0].shape[2]))     # r_0 != 1
        with pytest.raises((ValueError, qtt.QttError)):
            op.compressed_matvec(b6)
