"""Oracle implementations of the QTT matrix x dense vector product.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Independent of the CUDA
path: no shared kernels, layouts, helpers or constants.

Notation (PAPER.md; readings R1-R3 of DESIGN.md):
  cores[k-1] = G_k with shape (r_{k-1}, 2, 2, r_k), element G_k[a, i, j, b]
  = G_k(alpha_{k-1}=a, overline{i_k j_k}, alpha_k=b) with i_k the row (target)
  digit and j_k the column (source) digit.  Digits are LSB first:
  i = sum_k i_k 2^{k-1} (i_1 is the finest level).
  Dense vectors are arrays of shape (nrhs, N) (row s = right-hand side s).
"""
from __future__ import annotations

import numpy as np


def _ranks(cores):
    return [int(cores[0].shape[0])] + [int(G.shape[3]) for G in cores]


# ---------------------------------------------------------------------------
# The definition: Eq. (TTdeccores) applied to the product-tree
# tensorization of a matrix:
#   A(overline{i_1..i_d}, overline{j_1..j_d})
#     = G_1(:, i_1 j_1, :) G_2(:, i_2 j_2, :) ... G_d(:, i_d j_d, :)
# ---------------------------------------------------------------------------
def entry(cores, i: int, j: int, dtype=np.float64):
    """A(i, j) as the product of d core slices (Eq. TTdeccores; SPEC tt_entry S:76-84)."""
    v = np.ones((1, 1), dtype=dtype)
    for k, G in enumerate(cores):
        ik = (i >> k) & 1
        jk = (j >> k) & 1
        v = v @ G[:, ik, jk, :].astype(dtype)
    return v[0, 0]


def dense_matrix(cores, dtype=np.float64, guard: int = 1 << 24):
    """Materialise the N x N matrix A (brute force; SPEC tt_to_dense S:86-94).

    Contract the cores in order 1..d.  After k cores the partial tensor is
    T[I, J, alpha_k] over the k finest row/column digits; core k+1 adds the
    digit i_{k+1} (resp. j_{k+1}) as the new MOST significant row (column)
    digit.  Guard: N*N <= 2**24 scalars (N <= 4096), as SPEC S:88.
    """
    d = len(cores)
    N = 1 << d
    if N * N > guard:
        raise ValueError("dense_matrix: N*N exceeds the densify guard")
    T = cores[0][0].astype(dtype)                    # [i_1, j_1, alpha_1]
    for k in range(1, d):
        G = cores[k].astype(dtype)                   # [a, i, j, b]
        n = T.shape[0]
        T = np.einsum("IJa,aijb->iIjJb", T, G).reshape(2 * n, 2 * n, G.shape[3])
    return T[:, :, 0]


def apply_dense(cores, x, dtype=np.float64):
    """y = A x with A materialised (the definition; N <= 4096)."""
    A = dense_matrix(cores, dtype)
    x = np.atleast_2d(np.asarray(x, dtype=dtype))
    return x @ A.T


# ---------------------------------------------------------------------------
# Bitwise-position sweep (SURVEY §8(c) oracle 2).  Deliberately NOT the
# rotating layout of Alg. 2: the partial result keeps position p fixed and
# contracts one source digit per level in place.
#   T_0[p] = x[p];
#   T_k[p][b] = sum_{j,a} G_k[a, bit_{k-1}(p), j, b] * T_{k-1}[p with bit k-1 := j][a]
#   y[p] = T_d[p][0]
# After k levels, bits 0..k-1 of p are target digits i_1..i_k and bits
# k..d-1 are source digits j_{k+1}..j_d ("upward pass").
# ---------------------------------------------------------------------------
def apply_bitwise(cores, x, dtype=np.float64):
    x = np.atleast_2d(np.asarray(x, dtype=dtype))
    nrhs, N = x.shape
    d = len(cores)
    assert N == 1 << d
    p = np.arange(N, dtype=np.int64)
    out = np.empty((nrhs, N), dtype=dtype)
    for s in range(nrhs):
        T = x[s].reshape(N, 1)
        for k in range(d):
            G = cores[k].astype(dtype)
            bit = (p >> k) & 1
            Tn = np.zeros((N, G.shape[3]), dtype=dtype)
            for j in (0, 1):
                src = (p & ~(1 << k)) | (j << k)
                for i in (0, 1):
                    m = bit == i
                    Tn[m] += T[src[m]] @ G[:, i, j, :]
            T = Tn
        out[s] = T[:, 0]
    return out


# ---------------------------------------------------------------------------
# Alg. 2 (alg:TT-matvec), written in the paper's order and its
# Matlab (column-major) notation.  Bars are column-major: overline{a b} =
# a + (range of a) * b, so the first listed index is the fastest.
# ---------------------------------------------------------------------------
def alg2_sweep(cores, b, dtype=np.float64):
    """Run Alg. 2 lines 3-9 on one vector b; return y_d (r_d x N).

    Works for any r_d (an open right bond), which the chunked/sampled uses
    need; with r_d = 1 the result of Alg. 2 is y = y_d^T (line 10).
    """
    b = np.asarray(b, dtype=dtype).reshape(-1)
    N = b.shape[0]
    d = len(cores)
    assert N == 1 << d
    # line 3: y_0 = b^T with alpha_0 trivial (r_0 = 1)
    y = np.asfortranarray(b.reshape(1, N))
    for k in range(1, d + 1):
        G = cores[k - 1].astype(dtype)
        r_prev, r_k = G.shape[0], G.shape[3]
        # line 5: M_k(overline{alpha_k i_k}, overline{alpha_{k-1} j_k}) = G_k(alpha_{k-1}, overline{i_k j_k}, alpha_k)
        #   row alpha_k + r_k i_k, column alpha_{k-1} + r_{k-1} j_k
        M = np.empty((2 * r_k, 2 * r_prev), dtype=dtype)
        for i in (0, 1):
            for j in (0, 1):
                M[i * r_k:(i + 1) * r_k, j * r_prev:(j + 1) * r_prev] = G[:, i, j, :].T
        # line 6: b_k(overline{alpha_{k-1} j_k}, overline{J^BOX_k I^LCL_{k-1}}) = y_{k-1}(alpha_{k-1}, overline{J^BOX_{k-1} I^LCL_{k-1}})
        #   a column-major reshape (J^BOX_{k-1} = overline{j_k J^BOX_k}, j_k fastest)
        bk = np.reshape(y, (2 * r_prev, N // 2), order="F")
        # line 7: phi_k = M_k b_k
        phi = M @ bk
        # line 8: y_k(alpha_k, overline{J^BOX_k I^LCL_k}) = phi_k(overline{alpha_k i_k}, overline{J^BOX_k I^LCL_{k-1}})
        #   I^LCL_k = overline{I^LCL_{k-1} i_k}: i_k becomes the slowest column digit
        t = np.reshape(phi, (r_k, 2, N // 2), order="F")          # [alpha_k, i_k, c']
        y = np.reshape(np.transpose(t, (0, 2, 1)), (r_k, N), order="F")  # column c' + (N/2) i_k
        y = np.asfortranarray(y)
    return y


def apply_alg2(cores, x, dtype=np.float64):
    """y = A x by Alg. 2 (line 10: y = y_d^T), one RHS at a time."""
    x = np.atleast_2d(np.asarray(x, dtype=dtype))
    out = np.empty_like(x)
    for s in range(x.shape[0]):
        yd = alg2_sweep(cores, x[s], dtype)
        assert yd.shape[0] == 1
        out[s] = yd[0]
    return out


# ---------------------------------------------------------------------------
# Alg. 2 with BLAS calls and no copies (SURVEY §8(c) oracle 3, the timed CPU
# baseline).  The same lines 3-10 as ``alg2_sweep``; only the storage of y_k
# differs: Matlab keeps y_k (r_k x N) column-major, and a C-order numpy array
# Y_k of shape [N][r_k] is exactly those bytes, Y_k[c][alpha] = y_k(alpha, c).
#   line 6  b_k(overline{alpha_{k-1} j_k}, c') = y_{k-1}(alpha_{k-1}, overline{j_k c'})
#           -> b_k^T = Y_{k-1} viewed as [N/2][2 r_{k-1}]  (free reshape)
#   line 7  phi_k = M_k b_k  ->  phi_k^T = b_k^T M_k^T
#   line 8  y_k(alpha_k, overline{c' i_k}) = phi_k(overline{alpha_k i_k}, c')
#           -> Y_k[c' + (N/2) i_k] = (b_k^T M_k^T)[c', i_k r_k : (i_k+1) r_k]
# so each level is two matmuls, one per i_k, each writing straight into its
# half of Y_k (``out=``); two buffers rotate.
# ---------------------------------------------------------------------------
def _mt_half(G, i, dtype):
    """Columns i r_k .. (i+1) r_k - 1 of M_k^T (Alg. 2 line 5):
    M_k^T[alpha_{k-1} + r_{k-1} j, beta] = G_k[alpha_{k-1}, i, j, beta]."""
    Gi = np.asarray(G[:, i, :, :], dtype=dtype)              # [alpha_{k-1}, j, beta]
    return np.ascontiguousarray(Gi.transpose(1, 0, 2).reshape(2 * G.shape[0], G.shape[3]))


def blas_sweep(cores, b, dtype=np.float64):
    """Alg. 2 lines 3-9 on one vector b of length 2^len(cores); returns Y_d,
    the C-order [N][r_d] array (= y_d column-major; an open right bond r_d > 1
    is allowed, as ``alg2_sweep``).  With no cores, Y_0 = b as [N][1]."""
    b = np.ascontiguousarray(np.asarray(b, dtype=dtype).reshape(-1))
    N = b.shape[0]
    d = len(cores)
    assert N == 1 << d
    ranks = [1] + [int(G.shape[3]) for G in cores]
    if d == 0:
        return b.reshape(N, 1)
    rmax = max(ranks[1:])
    bufs = [np.empty(N * rmax, dtype=dtype), np.empty(N * rmax, dtype=dtype)]
    Y = b                                                      # line 3: y_0 = b^T (r_0 = 1)
    for k in range(1, d + 1):
        G = cores[k - 1]
        r_prev, r_k = ranks[k - 1], ranks[k]
        inp = Y.reshape(N // 2, 2 * r_prev)                    # line 6 (view)
        out = bufs[k % 2][: N * r_k].reshape(N, r_k)
        for i in (0, 1):                                       # lines 7-8
            np.matmul(inp, _mt_half(G, i, dtype), out=out[i * (N // 2):(i + 1) * (N // 2)])
        Y = out
    return Y.reshape(N, ranks[d])


def apply_blas_sweep(cores, x, dtype=np.float64):
    """y = A x by ``blas_sweep`` (line 10: y = y_d^T, r_d = 1), one RHS at a time."""
    x = np.atleast_2d(np.asarray(x, dtype=dtype))
    out = np.empty_like(x)
    for s in range(x.shape[0]):
        Y = blas_sweep(cores, x[s], dtype)
        assert Y.shape[1] == 1
        out[s] = Y[:, 0]
    return out


# ---------------------------------------------------------------------------
# Chunked sweep (SURVEY §8(c) oracle 4; top-bit blocks).  Split
# the index into its top s digits (g for the column, h for the row) and the
# low d - s digits.  By the definition (Eq. TTdeccores),
#   A(h n + i', g n + j') = [G_1 ... G_{d-s}](i', j') . c_{h,g},
#   c_{h,g} = G_{d-s+1}(:, h_1 g_1, :) ... G_d(:, h_s g_s, :)     (r_{d-s} x 1)
# so y[h-block] = sum_g T_g c_{h,g} with T_g = Alg. 2 levels 1..d-s applied
# to the block x[g-block] alone (Y_{d-s} of that block, open right bond).
# Peak memory is two n x r buffers (n = N / 2^s), which is what lets c5
# (N = 2^27, r = 24: 25.8 GB per full buffer) run on a modest host.
# ---------------------------------------------------------------------------
def top_projection(cores, s: int, h: int, g: int, dtype=np.float64):
    """c_{h,g} = prod_{l=1..s} G_{d-s+l}(:, h_l, g_l, :), an r_{d-s}-vector
    (h_l, g_l = bit l-1 of h, g)."""
    d = len(cores)
    c = np.eye(int(cores[d - s].shape[0]) if s else 1, dtype=dtype)
    for l in range(s):
        G = np.asarray(cores[d - s + l], dtype=dtype)
        c = c @ G[:, (h >> l) & 1, (g >> l) & 1, :]
    return c[:, 0]


def apply_chunked(cores, x, s: int, dtype=np.float64):
    """y = A x through 2^s top-bit blocks: Alg. 2 (``blas_sweep``) on each
    block of x for levels 1..d-s, then the projections onto every output block."""
    x = np.atleast_2d(np.asarray(x, dtype=dtype))
    nrhs, N = x.shape
    d = len(cores)
    assert N == 1 << d and 0 <= s <= d
    P, n = 1 << s, N >> s
    low = list(cores[: d - s])
    out = np.zeros((nrhs, N), dtype=dtype)
    for t in range(nrhs):
        for g in range(P):
            T = blas_sweep(low, x[t, g * n:(g + 1) * n], dtype)     # [n][r_{d-s}]
            for h in range(P):
                out[t, h * n:(h + 1) * n] += T @ top_projection(cores, s, h, g, dtype)
    return out


# ---------------------------------------------------------------------------
# Rank-1 (Kronecker) operators applied mode by mode: A = F_d (x) ... (x) F_1
# ("Kronecker product"; SURVEY §8(c) pin P3).  With x reshaped to
# (2,)*d in C order, axis 0 is digit d (MSB) and axis d-1 is digit 1 (LSB);
# F_k acts on axis d-k.  O(N d) work: a closed form at any d that shares
# nothing with Alg. 2.
# ---------------------------------------------------------------------------
def kron_apply_modes(factors, x, dtype=np.float64):
    x = np.atleast_2d(np.asarray(x, dtype=dtype))
    nrhs, N = x.shape
    d = len(factors)
    assert N == 1 << d
    out = np.empty_like(x)
    for t in range(nrhs):
        Z = x[t].reshape((2,) * d) if d else x[t].reshape(())
        for k, F in enumerate(factors, start=1):
            ax = d - k
            Z = np.moveaxis(np.tensordot(np.asarray(F, dtype=dtype), Z, axes=([1], [ax])), 0, ax)
        out[t] = np.reshape(Z, N)
    return out


# ---------------------------------------------------------------------------
# Sampled outputs: y[i] = sum_j A(i, j) x[j] for a few rows i, at any N.
# With the row digits fixed, contract the source digits j_1, j_2, ... in turn:
#   W_0[J, .] = x[J];  W_k[J', b] = sum_{j,a} W_{k-1}[j + 2 J', a] G_k[a, i_k, j, b]
#   y[i] = W_d[0, 0]
# This is Eq. (TTdeccores) summed over j in a different association from
# Alg. 2 (no rotation, no row separation).
# ---------------------------------------------------------------------------
def apply_rows(cores, x, rows, dtype=np.float64):
    x = np.atleast_2d(np.asarray(x, dtype=dtype))
    nrhs, N = x.shape
    rows = np.asarray(rows, dtype=np.int64)
    out = np.empty((nrhs, rows.size), dtype=dtype)
    for s in range(nrhs):
        for t, i in enumerate(rows):
            W = x[s].reshape(N, 1)
            for k, G in enumerate(cores):
                ik = (int(i) >> k) & 1
                n = W.shape[0] // 2
                W = W.reshape(n, 2, W.shape[1])      # [J', j, a]
                W = np.einsum("Jja,ajb->Jb", W, G[:, ik, :, :].astype(dtype), optimize=True)
            out[s, t] = W[0, 0]
    return out


# ---------------------------------------------------------------------------
# Operator algebra used by pins.
# ---------------------------------------------------------------------------
def compose(A_cores, B_cores):
    """Cores of the product A.B (P:1226-1231 rank-product argument; SPEC tt_matmat S:311-319).

    C_k[(a,a'), i, j, (b,b')] = sum_l G^A_k[a, i, l, b] G^B_k[a', l, j, b'].
    """
    out = []
    for GA, GB in zip(A_cores, B_cores):
        C = np.einsum("ailb,cljd->acijbd", GA, GB)
        ra, rb = GA.shape[0] * GB.shape[0], GA.shape[3] * GB.shape[3]
        out.append(C.reshape(ra, 2, 2, rb))
    return out


def transpose(cores):
    """Cores of A^T: swap the row and column digit of every core."""
    return [np.ascontiguousarray(G.transpose(0, 2, 1, 3)) for G in cores]


def kron_vector_cores(vs):
    """TT-vector cores (rank 1) of x = v_d (x) ... (x) v_1 (v_k has 2 entries)."""
    return [np.asarray(v, dtype=np.float64).reshape(1, 2, 1) for v in vs]


def compressed_matvec(A_cores, b_cores):
    """QTT-compressed matvec:
    G^c_k(overline{alpha beta}, i_k, overline{alpha' beta'})
      = sum_{j_k} G^A_k(alpha, overline{i_k j_k}, alpha') G^b_k(beta, j_k, beta').
    Returns TT-vector cores of c = A b (ranks r_A * r_b, no rounding)."""
    out = []
    for GA, Gb in zip(A_cores, b_cores):
        C = np.einsum("aijc,bjd->abicd", GA, Gb)
        out.append(C.reshape(GA.shape[0] * Gb.shape[0], 2, GA.shape[3] * Gb.shape[2]))
    return out


def tt_vector_entries(cores, idx, dtype=np.float64):
    """Entries v[i] = H_1(:, i_1, :) ... H_d(:, i_d, :) of a TT vector (Eq. TTdeccores)."""
    idx = np.asarray(idx, dtype=np.int64)
    out = np.empty(idx.size, dtype=dtype)
    for t, i in enumerate(idx):
        v = np.ones((1, 1), dtype=dtype)
        for k, H in enumerate(cores):
            v = v @ H[:, (int(i) >> k) & 1, :].astype(dtype)
        out[t] = v[0, 0]
    return out


def tt_vector_dense(cores, dtype=np.float64):
    """Dense N-vector of a TT vector with cores H_k (r_{k-1}, 2, r_k), LSB-first digits:
    v[overline{i_1..i_d}] = H_1(:, i_1, :) ... H_d(:, i_d, :)."""
    Z = cores[0][0].astype(dtype)                   # [i_1, alpha_1]
    for H in cores[1:]:
        H = H.astype(dtype)
        n = Z.shape[0]
        # new index i_{k} * n + I  (i_k most significant)
        Z = np.einsum("Ia,aib->iIb", Z, H).reshape(2 * n, H.shape[2])
    return Z[:, 0]
