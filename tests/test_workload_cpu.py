"""Seeded workload generators (host only): the structure they promise."""
import numpy as np

import oracle
from qtt_workload import bie_case


def test_bie_case_block_diagonal_m():
    """bie_case's M is block-diagonal over surfaces (PAPER Table 3's M):
    entries coupling two different surfaces (top index bits) vanish exactly; Y is dense."""
    d, pb = 8, 4
    rm, M, ry, Y, x = bie_case(3, d, pb, 12, 6, 2)
    assert rm == [min(2 ** k, 2 ** (d - k), 6) for k in range(d + 1)]
    assert ry == [min(2 ** k, 2 ** (d - k), 12) for k in range(d + 1)]
    A = oracle.dense_matrix(M)
    n = 1 << pb
    surf = np.arange(1 << d) // n
    off = surf[:, None] != surf[None, :]
    assert np.all(A[off] == 0.0)
    assert np.count_nonzero(A[~off]) > 0.9 * (~off).sum()
    assert np.count_nonzero(oracle.dense_matrix(Y)) > 0.99 * (1 << 2 * d)
    assert x.shape == (2, 1 << d)


def test_bie_case_is_seeded():
    a = bie_case(5, 6, 3, 4, 2, 1)
    b = bie_case(5, 6, 3, 4, 2, 1)
    for u, v in zip(a[1] + a[3] + [a[4]], b[1] + b[3] + [b[4]]):
        np.testing.assert_array_equal(u, v)
