"""Pins for the CPU oracle (-m "not gpu").

Each oracle function is checked against something other than itself: a
hand-worked golden example, closed forms evaluated by library routines
(np.roll, np.kron, scipy.linalg.hadamard), invariants (composition,
transpose, linearity), brute force, and a longdouble re-run.  A mutation test
at the end shows the pins catch the plausible mistakes (transposed core,
reversed digit order, dropped bond term).
"""
import numpy as np
import pytest
import scipy.linalg

import oracle
from oracle import qtt_oracle as Q
from qtt_workload import closed_forms as CF
from qtt_workload import generate, random_case, flops_per_apply

APPLIES = {
    "alg2": oracle.apply_alg2,
    "blas": oracle.apply_blas_sweep,
    "chunked1": lambda cores, x: oracle.apply_chunked(cores, x, min(1, len(cores))),
    "chunked3": lambda cores, x: oracle.apply_chunked(cores, x, min(3, len(cores))),
    "bitwise": oracle.apply_bitwise,
    "dense": oracle.apply_dense,
    "rows": lambda cores, x: oracle.apply_rows(cores, x, np.arange(np.atleast_2d(x).shape[1])),
}


def _golden_cores(g):
    r = [int(v) for v in g["ranks"]]
    G1 = np.array(g["G1"]).reshape(r[0], 2, 2, r[1])
    G2 = np.array(g["G2"]).reshape(r[1], 2, 2, r[2])
    return [G1, G2]


# --- golden (hand-worked, Eq. TTdeccores + P:953-962) ----------------------
def test_golden_tiny(golden):
    g = golden("tiny_d2_rank2.txt")
    cores = _golden_cores(g)
    A = np.array(g["A"]).reshape(4, 4)
    np.testing.assert_array_equal(oracle.dense_matrix(cores), A)
    for i in range(4):
        for j in range(4):
            assert oracle.entry(cores, i, j) == A[i, j]
    x = np.array(g["x"])
    for name, f in APPLIES.items():
        np.testing.assert_array_equal(f(cores, x)[0], np.array(g["y"]), err_msg=name)


# --- identity: exact -------------------------------------
@pytest.mark.parametrize("d", [1, 2, 5, 10])
def test_identity_exact(d):
    x = np.random.default_rng(d).standard_normal((2, 1 << d))
    cores = CF.identity_cores(d)
    for name, f in APPLIES.items():
        if name == "dense" and d > 12:
            continue
        np.testing.assert_array_equal(f(cores, x), x, err_msg=name)


# --- Kronecker of 2x2 factors: A = F_d (x) ... (x) F_1 (np.kron) -------------
@pytest.mark.parametrize("d", [1, 3, 6, 9])
def test_kronecker_dense_equals_np_kron(d):
    rng = np.random.default_rng(100 + d)
    F = [rng.standard_normal((2, 2)) for _ in range(d)]
    A = np.ones((1, 1))
    for Fk in F:              # F_1 innermost (fastest digit)
        A = np.kron(Fk, A)
    cores = CF.kron_cores(F)
    np.testing.assert_allclose(oracle.dense_matrix(cores), A, rtol=1e-13, atol=1e-14)
    x = rng.standard_normal((1, 1 << d))
    ref = x @ A.T
    for name, f in APPLIES.items():
        np.testing.assert_allclose(f(cores, x), ref, rtol=1e-12, atol=1e-12, err_msg=name)


def test_walsh_hadamard():
    d = 10
    H2 = np.array([[1.0, 1.0], [1.0, -1.0]])
    cores = CF.kron_cores([H2] * d)
    x = np.random.default_rng(7).standard_normal((1, 1 << d))
    ref = x @ scipy.linalg.hadamard(1 << d).T.astype(float)
    for name, f in APPLIES.items():
        np.testing.assert_allclose(f(cores, x), ref, rtol=0, atol=1e-10, err_msg=name)


def test_diagonal_scaling():
    d = 8
    rng = np.random.default_rng(8)
    diags = [rng.uniform(0.5, 2.0, 2) for _ in range(d)]
    cores = CF.kron_cores([np.diag(v) for v in diags])
    p = np.arange(1 << d)
    scale = np.ones(1 << d)
    for k, v in enumerate(diags):
        scale *= v[(p >> k) & 1]
    x = rng.standard_normal((1, 1 << d))
    for name, f in APPLIES.items():
        np.testing.assert_allclose(f(cores, x)[0], scale * x[0], rtol=1e-14, err_msg=name)


# --- cyclic shift (rank 2, exact): y == np.roll(x, s) bitwise -----------------
@pytest.mark.parametrize("d,s", [(1, 1), (2, 1), (3, 5), (6, 1), (8, 255), (10, 1), (10, 333)])
def test_shift_exact(d, s):
    x = np.random.default_rng(s).standard_normal((1, 1 << d))
    cores = CF.shift_cores(d, s)
    assert max(CF.ranks_of(cores)) <= 2
    for name, f in APPLIES.items():
        if name == "dense" and d > 12:
            continue
        np.testing.assert_array_equal(f(cores, x)[0], np.roll(x[0], s), err_msg=name)


# --- random operators: four independent evaluations agree ---------------------
@pytest.mark.parametrize("seed,d,maxr,nrhs", [(1, 1, 1, 1), (2, 4, 3, 2), (3, 7, 6, 1), (4, 9, 8, 3), (5, 11, 5, 1)])
def test_random_all_variants_agree(seed, d, maxr, nrhs):
    ranks, cores, x = random_case(seed, d, maxr, nrhs)
    ref = oracle.apply_dense(cores, x)
    for name, f in APPLIES.items():
        oracle.assert_close(f(cores, x), ref, l2_tol=1e-13)
    # spot entries from the product of slices
    rng = np.random.default_rng(seed)
    A = oracle.dense_matrix(cores)
    for _ in range(10):
        i, j = rng.integers(0, 1 << d, 2)
        assert abs(oracle.entry(cores, int(i), int(j)) - A[i, j]) <= 1e-13 * (1 + abs(A[i, j]))


# --- column / entry pin: x = e_j gives column j of A ----------------------------
def test_unit_vector_gives_column():
    ranks, cores, _ = random_case(11, 8, 5)
    N = 1 << 8
    for j in (0, 1, 77, N - 1):
        e = np.zeros((1, N))
        e[0, j] = 1.0
        col = np.array([oracle.entry(cores, i, j) for i in range(N)])
        np.testing.assert_allclose(oracle.apply_alg2(cores, e)[0], col, rtol=1e-12, atol=1e-15)


# --- composition: apply(AB) = apply(A, apply(B)) -------
def test_composition():
    _, A, x = random_case(21, 10, 4)
    _, B, _ = random_case(22, 10, 3)
    AB = oracle.compose(A, B)
    ra, rb = CF.ranks_of(A), CF.ranks_of(B)
    assert CF.ranks_of(AB) == [p * q for p, q in zip(ra, rb)]   # rank-product law
    lhs = oracle.apply_alg2(AB, x)
    rhs = oracle.apply_alg2(A, oracle.apply_alg2(B, x))
    oracle.assert_close(lhs, rhs, l2_tol=1e-13)
    # shift composed with itself is shift by 2
    S1 = CF.shift_cores(10, 1)
    np.testing.assert_array_equal(oracle.apply_alg2(oracle.compose(S1, S1), x)[0], np.roll(x[0], 2))


# --- transpose and linearity ------------------------------------------------------
def test_transpose_and_linearity():
    d = 10
    _, A, x = random_case(31, d, 6, nrhs=2)
    rng = np.random.default_rng(32)
    u = rng.standard_normal(1 << d)
    lhs = u @ oracle.apply_alg2(A, x[0])[0]
    rhs = oracle.apply_alg2(oracle.transpose(A), u)[0] @ x[0]
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(u) * np.linalg.norm(x[0])
    a, b = 0.7, -1.3
    y = oracle.apply_alg2(A, a * x[0] + b * x[1])[0]
    y2 = a * oracle.apply_alg2(A, x[0])[0] + b * oracle.apply_alg2(A, x[1])[0]
    np.testing.assert_allclose(y, y2, rtol=0, atol=1e-12 * np.abs(y2).max())
    # transpose of shift(+1) is shift(-1)
    St = oracle.transpose(CF.shift_cores(d, 1))
    np.testing.assert_array_equal(oracle.apply_alg2(St, x[0])[0], np.roll(x[0], -1))


# --- Kronecker vector through the compressed matvec -----------------
@pytest.mark.parametrize("d,maxr", [(8, 5), (14, 8)])
def test_kron_vector_compressed_path(d, maxr):
    ranks, cores, _ = random_case(41 + d, d, maxr)
    rng = np.random.default_rng(d)
    vs = [rng.standard_normal(2) for _ in range(d)]
    xk = oracle.tt_vector_dense(oracle.kron_vector_cores(vs))
    # the Kronecker vector itself against np.kron (v_1 fastest)
    ref_x = np.ones(1)
    for v in vs:
        ref_x = np.kron(v, ref_x)
    np.testing.assert_allclose(xk, ref_x, rtol=1e-14)
    cc = oracle.compressed_matvec(cores, oracle.kron_vector_cores(vs))
    yc = oracle.tt_vector_dense(cc)
    oracle.assert_close(oracle.apply_alg2(cores, xk), yc[None, :], l2_tol=1e-13)
    idx = rng.integers(0, 1 << d, 20)
    np.testing.assert_allclose(oracle.tt_vector_entries(cc, idx), yc[idx], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(oracle.tt_vector_entries(oracle.kron_vector_cores(vs), idx), ref_x[idx], rtol=1e-14)


# --- c1: oracle against the dense 4096 x 4096 matvec (BASELINE.json configs[0]) ---
def test_c1_dense_materialised():
    cfg, cores, x = generate("c1")
    ref = oracle.apply_dense(cores, x)
    y = oracle.apply_alg2(cores, x)
    oracle.assert_close(y, ref, l2_tol=1e-13)
    oracle.assert_close(oracle.apply_bitwise(cores, x), ref, l2_tol=1e-13)
    rows = np.random.default_rng(0).integers(0, cfg.N, 64)
    oracle.assert_close(oracle.apply_rows(cores, x, rows), ref[:, rows], rms=np.linalg.norm(ref) / np.sqrt(cfg.N))


# --- P10: the fp64 oracle against a longdouble run ----------------------------------
def test_longdouble_precision_c2():
    cfg, cores, x = generate("c2")
    y64 = oracle.apply_alg2(cores, x)
    yld = oracle.apply_alg2(cores, x, dtype=np.longdouble)
    m = oracle.compare(y64, yld.astype(np.float64))[0]
    assert m["rel_l2"] < 1e-14, m
    assert m["elem_floor"] < 1e-13, m


# --- Alg. 2 with an open right bond: top-bit chunk decomposition -------
def test_open_bond_chunks():
    d, s = 10, 2
    ranks, cores, x = random_case(51, d, 5)
    P = 1 << s
    n = (1 << d) // P
    y = np.zeros(1 << d)
    for g in range(P):
        T = oracle.alg2_sweep(cores[: d - s], x[0, g * n:(g + 1) * n])   # r_{d-s} x n
        for h in range(P):
            c = np.eye(ranks[d - s])
            for l in range(s):
                c = c @ cores[d - s + l][:, (h >> l) & 1, (g >> l) & 1, :]
            # c_{h,g} = prod_l G_{d-s+l}[:, h_l, g_l, :]  (an r_{d-s} x 1 column)
            y[h * n:(h + 1) * n] += (c[:, 0] @ T)
    oracle.assert_close(y[None], oracle.apply_dense(cores, x), l2_tol=1e-13)


# --- generator properties ---------------------------------------------------------------
def test_generator_c3x16_column0_and_flops():
    _, c3, x1 = generate("c3", with_x=True)
    _, c3b, x16 = generate("c3x16", with_x=True)
    for a, b in zip(c3, c3b):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(x16[0], x1[0])
    assert flops_per_apply(generate("c4", with_x=False)[0].ranks) == 4 * 32084 * (1 << 24)


# --- checker semantics ---------------------------------------------------------------------
def test_checker_floor_semantics():
    y = np.array([[1.0, -1.0, 1e-12, 2.0]])
    yh = y.copy()
    yh[0, 2] += 1e-15        # raw relative 1e-3 at a near-zero entry, tiny vs RMS
    m = oracle.compare(yh, y)[0]
    assert m["raw_offenders"] == 1 and m["elem_floor"] < 1e-14
    oracle.assert_close(yh, y)
    yh[0, 3] *= 1 + 1e-9
    with pytest.raises(AssertionError):
        oracle.assert_close(yh, y)


# --- mutation test: the pins catch plausible mistakes ----------------------------------------
def _mut_transposed(cores, x):
    return oracle.apply_alg2([G.transpose(0, 2, 1, 3) for G in cores], x)


def _mut_reversed_digits(cores, x):
    # treat core 1 as acting on the MSB
    d = len(cores)
    rev = [G.transpose(3, 1, 2, 0) for G in cores[::-1]]
    return oracle.apply_alg2(rev, x)


def _mut_dropped_bond(cores, x):
    cut = [G.copy() for G in cores]
    for G in cut[1:]:
        G[-1] = 0.0 if G.shape[0] > 1 else G[-1]
    return oracle.apply_alg2(cut, x)


@pytest.mark.parametrize("mut", [_mut_transposed, _mut_reversed_digits, _mut_dropped_bond])
def test_pins_catch_mutations(mut):
    d = 6
    x = np.random.default_rng(3).standard_normal((1, 1 << d))
    caught = False
    if not np.array_equal(mut(CF.shift_cores(d, 1), x)[0], np.roll(x[0], 1)):
        caught = True
    rng = np.random.default_rng(5)
    F = [rng.standard_normal((2, 2)) for _ in range(d)]
    A = np.ones((1, 1))
    for Fk in F:
        A = np.kron(Fk, A)
    if not np.allclose(mut(CF.kron_cores(F), x), x @ A.T, rtol=1e-12):
        caught = True
    assert caught


# --- Morton ordering (rem:interlace P:855-870; R18) ----
def test_morton_spec_example():
    # coordinate bits x=(1,0,0), y=(0,1,0), z=(0,0,1) (finest first)
    # i.e. x=1, y=2, z=4 -> digits interleave x,y,z per level: q bits
    # 0 (x_0)=1, 4 (y_1)=1, 8 (z_2)=1
    from oracle import morton as M
    assert M.morton_coords((1 << 0) | (1 << 4) | (1 << 8), 3, 3) == (1, 2, 4)
    assert M.natural_index((1, 2, 4), 3) == 1 + 8 * 2 + 64 * 4


@pytest.mark.parametrize("dim,levels", [(1, 5), (2, 3), (3, 2), (3, 3), (2, 5)])
def test_morton_bijection_and_bisection(dim, levels):
    """Bijection; and every aligned run of 2^(dim*l) consecutive QTT indices is
    an axis-aligned cube of side 2^l (the successive-bisection partition)."""
    from oracle import morton as M
    N = 1 << (dim * levels)
    p = M.morton_perm(dim, levels)
    assert sorted(p.tolist()) == list(range(N))
    n = 1 << levels
    coords = np.array(np.unravel_index(p, (n,) * dim)).T[:, ::-1]   # (x, y, z) of each q
    for l in range(levels + 1):
        run = 1 << (dim * l)
        for start in range(0, N, run):
            blk = coords[start:start + run]
            lo = blk.min(axis=0)
            assert np.all(blk.max(axis=0) - lo == (1 << l) - 1)
            assert np.all(lo % (1 << l) == 0)


def test_morton_dim1_identity_and_roundtrip():
    from oracle import morton as M
    assert np.array_equal(M.morton_perm(1, 6), np.arange(64))
    g = np.random.default_rng(0).standard_normal((2, 512))
    assert np.array_equal(M.unpack(M.pack(g, 3, 3), 3, 3), g)


def test_morton_separable_function():
    """A separable grid function f(x) g(y) h(z) packs to the Kronecker vector
    h (x) g (x) f in QTT digit order: digit dim*l + a of q selects bit l of axis a."""
    from oracle import morton as M
    rng = np.random.default_rng(1)
    lv = 3
    n = 1 << lv
    # small integers: every product is exact, so the check is bitwise
    f, g, h = (rng.integers(-9, 10, n).astype(float) for _ in range(3))
    grid = np.einsum("z,y,x->zyx", h, g, f).reshape(1, -1)
    xq = M.pack(grid, 3, lv)[0]
    for q in range(1 << (3 * lv)):
        x = sum(((q >> (3 * l)) & 1) << l for l in range(lv))
        y = sum(((q >> (3 * l + 1)) & 1) << l for l in range(lv))
        z = sum(((q >> (3 * l + 2)) & 1) << l for l in range(lv))
        assert xq[q] == f[x] * g[y] * h[z]


# --- the BLAS sweep and the chunked sweep: their own plausible mistakes are caught ----------
def _pins_hold(apply_fn):
    """True iff every pin below holds for ``apply_fn``: shift bitwise (np.roll),
    Kronecker against np.kron, and a random rank profile against the dense matrix."""
    d = 6
    x = np.random.default_rng(3).standard_normal((1, 1 << d))
    if not np.array_equal(apply_fn(CF.shift_cores(d, 5), x)[0], np.roll(x[0], 5)):
        return False
    rng = np.random.default_rng(5)
    F = [rng.standard_normal((2, 2)) for _ in range(d)]
    A = np.ones((1, 1))
    for Fk in F:
        A = np.kron(Fk, A)
    if not np.allclose(apply_fn(CF.kron_cores(F), x), x @ A.T, rtol=1e-12, atol=1e-13):
        return False
    _, cores, xr = random_case(9, d, 4)
    return bool(np.allclose(apply_fn(cores, xr), oracle.apply_dense(cores, xr), rtol=1e-12, atol=1e-13))


_orig_mt_half = Q._mt_half
_orig_top = Q.top_projection


def _mut_mt_swap_ij(G, i, dtype):
    return _orig_mt_half(np.ascontiguousarray(G.transpose(0, 2, 1, 3)), i, dtype)


def _mut_mt_merge_order(G, i, dtype):          # column merge as j + 2 alpha instead of alpha + r j
    return np.ascontiguousarray(np.asarray(G[:, i, :, :], dtype=dtype).reshape(2 * G.shape[0], G.shape[3]))


def _mut_top_swap_hg(cores, s, h, g, dtype=np.float64):
    return _orig_top(cores, s, g, h, dtype)


def _mut_top_msb_first(cores, s, h, g, dtype=np.float64):
    rev = lambda v: sum(((v >> l) & 1) << (s - 1 - l) for l in range(s))
    return _orig_top(cores, s, rev(h), rev(g), dtype)


@pytest.mark.parametrize("name,mut,fn", [
    ("_mt_half", _mut_mt_swap_ij, "blas"),
    ("_mt_half", _mut_mt_merge_order, "blas"),
    ("top_projection", _mut_top_swap_hg, "chunked3"),
    ("top_projection", _mut_top_msb_first, "chunked3"),
])
def test_pins_catch_sweep_mutations(monkeypatch, name, mut, fn):
    assert _pins_hold(APPLIES[fn])
    monkeypatch.setattr(Q, name, mut)
    assert not _pins_hold(APPLIES[fn])


@pytest.mark.parametrize("d,s", [(5, 0), (5, 2), (5, 5), (9, 4), (12, 3)])
def test_chunked_equals_alg2_dense(d, s):
    _, cores, x = random_case(60 + d + s, d, 6, nrhs=2)
    ref = oracle.apply_dense(cores, x)
    oracle.assert_close(oracle.apply_chunked(cores, x, s), ref, l2_tol=1e-13)
    oracle.assert_close(oracle.apply_blas_sweep(cores, x), ref, l2_tol=1e-13)


# --- Kronecker operators applied mode by mode (P3 at any d) --------------------------------
@pytest.mark.parametrize("d", [0, 1, 4, 7, 10])
def test_kron_modes_equals_np_kron(d):
    rng = np.random.default_rng(200 + d)
    F = [rng.standard_normal((2, 2)) for _ in range(d)]
    A = np.ones((1, 1))
    for Fk in F:              # F_1 innermost (fastest digit)
        A = np.kron(Fk, A)
    x = rng.standard_normal((2, 1 << d))
    np.testing.assert_allclose(oracle.kron_apply_modes(F, x), x @ A.T, rtol=1e-12, atol=1e-13)


def test_kron_modes_hadamard_and_permutation():
    d = 11
    H2 = np.array([[1.0, 1.0], [1.0, -1.0]])
    x = np.random.default_rng(4).integers(-5, 6, (1, 1 << d)).astype(float)
    # integer data: the Walsh-Hadamard transform is exact, compare bitwise
    np.testing.assert_array_equal(oracle.kron_apply_modes([H2] * d, x),
                                  x @ scipy.linalg.hadamard(1 << d).T.astype(float))
    # swap matrix on digit k only: y[i] = x[i xor 2^(k-1)]
    X2 = np.array([[0.0, 1.0], [1.0, 0.0]])
    for k in (1, 5, d):
        F = [np.eye(2)] * d
        F = F[:k - 1] + [X2] + F[k:]
        np.testing.assert_array_equal(oracle.kron_apply_modes(F, x)[0], x[0][np.arange(1 << d) ^ (1 << (k - 1))])


def test_kron_modes_agrees_with_sweeps_large():
    d = 16
    rng = np.random.default_rng(17)
    F = [rng.standard_normal((2, 2)) / 1.3 for _ in range(d)]
    x = rng.standard_normal((1, 1 << d))
    ref = oracle.kron_apply_modes(F, x)
    cores = CF.kron_cores(F)
    oracle.assert_close(oracle.apply_blas_sweep(cores, x), ref, l2_tol=1e-13)
    oracle.assert_close(oracle.apply_chunked(cores, x, 4), ref, l2_tol=1e-13)


# --- TT vectors of rank > 1: an exact closed form, and the compressed matvec ----------------
def _linear_tt(d, a, b):
    """Exact rank-2 TT vector of v[i] = a + b i (i = sum_k i_k 2^{k-1}): the bond
    carries (running sum, 1)."""
    cores = []
    for k in range(d):
        w = float(b) * (1 << k)
        if d == 1:
            H = np.array([[[a], [a + w]]])                       # (1, 2, 1)
        elif k == 0:
            H = np.zeros((1, 2, 2))
            for i in (0, 1):
                H[0, i] = [1.0, a + w * i]
        elif k == d - 1:
            H = np.zeros((2, 2, 1))
            for i in (0, 1):
                H[:, i, 0] = [w * i, 1.0]
        else:
            H = np.zeros((2, 2, 2))
            for i in (0, 1):
                H[:, i, :] = [[1.0, w * i], [0.0, 1.0]]
        cores.append(H)
    return cores


@pytest.mark.parametrize("d", [1, 2, 9])
def test_tt_vector_linear_closed_form(d):
    cores = _linear_tt(d, 3.0, -2.0)
    ref = 3.0 - 2.0 * np.arange(1 << d, dtype=float)
    np.testing.assert_array_equal(oracle.tt_vector_dense(cores), ref)
    idx = np.arange(1 << d)
    np.testing.assert_array_equal(oracle.tt_vector_entries(cores, idx), ref)


def _mut_compressed_right_bond(A_cores, b_cores):
    out = []
    for GA, Gb in zip(A_cores, b_cores):
        C = np.einsum("aijc,bjd->abidc", GA, Gb)       # right bond merged as (beta', alpha')
        out.append(C.reshape(GA.shape[0] * Gb.shape[0], 2, GA.shape[3] * Gb.shape[2]))
    return out


@pytest.mark.parametrize("seed,d,ra,rb", [(1, 8, 5, 2), (2, 9, 4, 4), (3, 7, 3, 6)])
def test_compressed_matvec_rank_gt1(seed, d, ra, rb):
    """c = A b in QTT form for a TT vector b of rank up to rb > 1:
    its dense form equals Alg. 2 applied to the dense b; the (beta', alpha')
    mutant of the right-bond merge fails the same check."""
    from qtt_workload import random_tt_vector
    _, A, _ = random_case(seed, d, ra)
    _, bc = random_tt_vector(seed + 50, d, rb)
    assert max(H.shape[2] for H in bc[:-1]) > 1
    bdense = oracle.tt_vector_dense(bc)
    ref = oracle.apply_dense(A, bdense)
    oracle.assert_close(oracle.tt_vector_dense(oracle.compressed_matvec(A, bc))[None], ref, l2_tol=1e-13)
    m = oracle.compare(oracle.tt_vector_dense(_mut_compressed_right_bond(A, bc))[None], ref)[0]
    assert m["rel_l2"] > 1e-3
    # the linear vector: A (a + b i) computed through the compressed matvec
    lin = _linear_tt(d, 0.5, 0.25)
    oracle.assert_close(oracle.tt_vector_dense(oracle.compressed_matvec(A, lin))[None],
                        oracle.apply_dense(A, 0.5 + 0.25 * np.arange(1 << d)), l2_tol=1e-13)
