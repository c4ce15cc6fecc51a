"""QTT cores of operators whose action has a closed form (test pins).

These build inputs only; the expected results are computed in the tests by
library routines (``np.roll``, ``np.kron``, ``scipy.linalg.hadamard``) that
share nothing with either the oracle or the CUDA path.

* identity   (SPEC S:271-279 ``tt_identity``; "a Kronecker
  product of identities"): all ranks 1, G_k[0,i,j,0] = delta_ij.
* Kronecker  (rank 1): G_k[0,:,:,0] = F_k gives A = F_d (x) ... (x) F_1 under
  the LSB-first digit convention (row index i = sum_k i_k 2^{k-1}).
* cyclic shift by s (rank 2, exact): binary addition i = j + s (mod N) as a
  carry chain from the least significant digit; the bond index is the carry.
"""
from __future__ import annotations

import numpy as np


def identity_cores(d: int):
    return [np.eye(2).reshape(1, 2, 2, 1).copy() for _ in range(d)]


def kron_cores(factors):
    """factors[k] is the 2x2 matrix F_{k+1}[i, j] of level k+1 (row digit i)."""
    return [np.asarray(F, dtype=np.float64).reshape(1, 2, 2, 1).copy() for F in factors]


def shift_cores(d: int, s: int = 1):
    """Cores of the cyclic shift (A x)[i] = x[(i - s) mod N], i.e. np.roll(x, s).

    A(i, j) = 1 iff i = (j + s) mod N.  Level k adds the digit s_k of s and the
    incoming carry c to j_k: i_k = (j_k + s_k + c) mod 2, carry out
    c' = (j_k + s_k + c) >= 2.  The level-1 carry-in is 0 (r_0 = 1) and the
    carry out of level d is dropped (mod N), so r_d = 1.
    """
    N = 1 << d
    s %= N
    cores = []
    for k in range(d):
        sk = (s >> k) & 1
        cin = [0] if k == 0 else [0, 1]
        rl = len(cin)
        last = k == d - 1
        rr = 1 if last else 2
        G = np.zeros((rl, 2, 2, rr))
        for a, c in enumerate(cin):
            for j in range(2):
                t = j + sk + c
                i, cout = t & 1, t >> 1
                b = 0 if last else cout
                G[a, i, j, b] = 1.0
        cores.append(G)
    return cores


def ranks_of(cores):
    return [int(cores[0].shape[0])] + [int(G.shape[3]) for G in cores]
