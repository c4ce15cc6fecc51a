"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star; reading R11): relative l2
<= 1e-12 per RHS column and elementwise relative error with an RMS floor
<= 1e-10; closed forms (identity, shift) bitwise.  Inputs come only from
``qtt_workload``; expected values only from ``oracle`` or library routines.
"""
import numpy as np
import pytest

import oracle
from qtt_workload import closed_forms as CF
from qtt_workload import generate, random_case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qtt():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    import paper_1511_06029_b200 as q
    q._lib.load()
    return q


def _per_stage(q, *a, **k):
    """An operator whose applies run the per-stage plan: these tests exercise
    the stage kernels (the fused one-launch apply has tests/test_gpu_fused.py)."""
    k.setdefault("fused", False)
    return q.QttOperator(*a, **k)


def gpu_apply(q, cores, x, max_stage_levels=None, **kw):
    op = _per_stage(q, cores, max_stage_levels=max_stage_levels)
    try:
        xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
        y = op.apply(xt, **kw)
        torch.cuda.synchronize()
        return y.cpu().numpy(), op.stages()
    finally:
        op.close()


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("d", [1, 2, 3, 5, 12, 20])
def test_identity_bitwise(qtt, d):
    x = np.random.default_rng(d).standard_normal((2, 1 << d))
    y, _ = gpu_apply(qtt, CF.identity_cores(d), x)
    np.testing.assert_array_equal(y, x)


@pytest.mark.parametrize("d,s", [(1, 1), (2, 3), (6, 1), (13, 1), (13, 4097), (21, 12345)])
def test_shift_bitwise(qtt, d, s):
    x = np.random.default_rng(s).standard_normal((1, 1 << d))
    y, _ = gpu_apply(qtt, CF.shift_cores(d, s), x)
    np.testing.assert_array_equal(y[0], np.roll(x[0], s))


def test_transposed_shift_bitwise(qtt):
    d = 16
    x = np.random.default_rng(0).standard_normal((1, 1 << d))
    y, _ = gpu_apply(qtt, oracle.transpose(CF.shift_cores(d, 1)), x)
    np.testing.assert_array_equal(y[0], np.roll(x[0], -1))


def test_kronecker_np_kron(qtt):
    d = 11
    rng = np.random.default_rng(3)
    F = [rng.standard_normal((2, 2)) for _ in range(d)]
    A = np.ones((1, 1))
    for Fk in F:
        A = np.kron(Fk, A)
    x = rng.standard_normal((2, 1 << d))
    y, _ = gpu_apply(qtt, CF.kron_cores(F), x)
    oracle.assert_close(y, x @ A.T)


# ------------------------------------------------------------------ random profiles
RANDOM_CASES = [
    # seed, d, max_rank, nrhs  (odd / non-multiple-of-8 ranks, ragged tails, tiny N)
    (1, 1, 1, 1), (2, 2, 2, 5), (3, 3, 4, 37), (4, 6, 7, 3), (5, 9, 13, 2), (6, 10, 24, 1),
    (7, 12, 33, 1), (8, 13, 48, 2), (9, 14, 5, 4), (10, 16, 17, 1), (11, 17, 31, 1), (12, 18, 3, 2),
    (13, 11, 64, 1), (14, 9, 100, 1),
]


@pytest.mark.parametrize("seed,d,maxr,nrhs", RANDOM_CASES)
def test_random_profiles(qtt, seed, d, maxr, nrhs):
    ranks, cores, x = random_case(seed, d, maxr, nrhs)
    y, _ = gpu_apply(qtt, cores, x)
    ref = oracle.apply_alg2(cores, x)
    oracle.assert_close(y, ref)


@pytest.mark.parametrize("r", [1, 2, 3, 8, 9, 16, 23, 32, 47, 48])
def test_constant_rank_sweep(qtt, r):
    ranks = [1] + [r] * 9 + [1]
    _, cores, x = random_case(100 + r, 10, r, 2, ranks=ranks)
    y, stages = gpu_apply(qtt, cores, x)
    oracle.assert_close(y, oracle.apply_alg2(cores, x))
    assert all(s["variant"] != "generic" for s in stages), stages


@pytest.mark.parametrize("maxL", [1, 6])
def test_generic_path_large_rank(qtt, maxL):
    # r = 1501: the 3002 x 3002 super-core of level 3 exceeds the wide kernel's 64 MiB -> generic
    ranks = [1, 2, 1501, 1501, 2, 1]
    _, cores, x = random_case(77, 5, 1501, 2, ranks=ranks)
    y, stages = gpu_apply(qtt, cores, x, max_stage_levels=maxL)
    if maxL == 1:
        assert any(s["variant"] == "generic" for s in stages)
    oracle.assert_close(y, oracle.apply_alg2(cores, x))


# ------------------------------------------------------------------ large ranks (NEXT-4: r up to 256)
@pytest.mark.parametrize("r", [56, 64, 96, 128, 200, 256])
@pytest.mark.parametrize("maxL", [1, None])
def test_large_rank_path(qtt, r, maxL):
    """Ranks above the smem-resident instances run on the wide (streamed
    super-core) kernel, one level per launch (maxL=1) or merged; never the
    generic kernel up to r = 256."""
    d = 11
    ranks = [1] + [r] * (d - 1) + [1]
    _, cores, x = random_case(1000 + r, d, r, 2, ranks=ranks)
    y, stages = gpu_apply(qtt, cores, x, max_stage_levels=maxL)
    assert all(s["variant"] != "generic" for s in stages), stages
    oracle.assert_close(y, oracle.apply_alg2(cores, x))


# ------------------------------------------------------------------ split-K wide stages
SPLIT_CASES = [
    # d, r, nrhs: constant rank, so the last stage's super-core has K = 2^L r
    # against few GEMM rows and the stage runs split-K (ragged last k-range
    # where S does not divide the chunk count)
    (17, 128, 1), (16, 192, 2), (18, 64, 1),
]


@pytest.mark.parametrize("d,r,nrhs", SPLIT_CASES)
def test_split_k_stages(qtt, d, r, nrhs):
    ranks = [1] + [r] * (d - 1) + [1]
    _, cores, x = random_case(5000 + 7 * d + r, d, r, nrhs, ranks=ranks)
    op = _per_stage(qtt, cores)
    try:
        splits = op.stage_splits(nrhs)
        assert max(splits) > 1, (op.stages(), splits)
        xt = torch.from_numpy(x).cuda()
        y1 = op.apply(xt)
        y2 = op.apply(xt)           # split counters left at zero; fixed-order sums
        ws = torch.empty(op.workspace_size(nrhs) // 8 + 1, dtype=torch.float64, device="cuda")
        y3 = torch.empty_like(xt)
        op.apply(xt, out=y3, workspace=ws)
        torch.cuda.synchronize()
        y1, y2, y3 = y1.cpu().numpy(), y2.cpu().numpy(), y3.cpu().numpy()
    finally:
        op.close()
    oracle.assert_close(y1, oracle.apply_alg2(cores, x))
    np.testing.assert_array_equal(y1, y2)
    np.testing.assert_array_equal(y1, y3)


def test_repeated_applies_alternating_inputs_bitwise(qtt):
    """Race check (found the early-PDL-trigger bug): c3, whose
    last stage runs split-K behind a PDL launch, applied 40 times to two
    alternating inputs; every result bitwise equal to the first of its input."""
    cfg, cores, x = generate("c3")
    x2 = np.ascontiguousarray(x[:, ::-1])
    with _per_stage(qtt, cores) as op:
        assert max(op.stage_splits(1)) > 1
        xs = [torch.from_numpy(x).cuda(), torch.from_numpy(x2).cuda()]
        refs = [op.apply(v).clone() for v in xs]
        torch.cuda.synchronize()
        bad = []
        for i in range(40):
            y = op.apply(xs[i % 2])
            torch.cuda.synchronize()
            if not torch.equal(y, refs[i % 2]):
                bad.append((i, int((y != refs[i % 2]).sum())))
    assert not bad, bad
    oracle.assert_close(refs[0].cpu().numpy(), oracle.apply_alg2(cores, x))


def test_repeated_applies_split_stage_bie_y(qtt):
    """Race check for split-K at scale (found the in-kernel reduction bug,
    DESIGN.md 6.8): the BIE factor Y (last stage K = 24320, split 4), pairs of
    applies enqueued back to back with alternating inputs, 100 times."""
    from qtt_workload import bie_case
    _, _, _, Y, x = bie_case(0, 21, 9, 95, 50, 1)
    x2 = np.ascontiguousarray(x[:, ::-1])
    with _per_stage(qtt, Y) as op:
        assert max(op.stage_splits(1)) > 1
        xs = [torch.from_numpy(v).cuda() for v in (x, x2)]
        refs = [op.apply(v).clone() for v in xs]
        torch.cuda.synchronize()
        bad = []
        for i in range(100):
            ys = [op.apply(v) for v in xs]
            torch.cuda.synchronize()
            bad += [(i, j) for j in range(2) if not torch.equal(ys[j], refs[j])]
    assert not bad, bad


def test_split_k_matches_unsplit_host_path(qtt):
    """qtt_apply_host's pipelined path never splits (its hooks need whole
    tiles); its result agrees with the split device path within tolerance."""
    d, r = 18, 64
    ranks = [1] + [r] * (d - 1) + [1]
    _, cores, x = random_case(6061, d, r, 1, ranks=ranks)
    with _per_stage(qtt, cores) as op:
        assert max(op.stage_splits(1)) > 1
        yd = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        yh = op.apply_host(x)
    oracle.assert_close(yd, yh)


# ------------------------------------------------------------------ diagonal (block-diagonal) levels
DIAG_CASES = [
    # d, max rank, nrhs, 0-based cores made diagonal in (i, j), the planner must pick "diag"
    (12, 6, 1, list(range(5, 12)), True),           # block-diagonal in the top 7 digits, r_d = 1
    (13, 8, 2, [4, 5, 6, 7], True),                 # a diagonal run in the middle (r_out <= 8 there)
    (11, 5, 3, [0, 1, 2], False),                   # the bottom digits
    (10, 4, 1, list(range(10)), True),              # every level: one diagonal stage
    (16, 3, 2, list(range(16)), True),              # a diagonal matrix: M = nrhs GEMM rows (lanes over ii)
    (15, 8, 1, list(range(3, 15)), True),           # 12 diagonal levels: M = 8 rows
    (14, 40, 2, [0, 1, 2, 3, 4], False),            # bottom digits at larger rank (parity only)
    (13, 64, 1, [5, 6], False),                     # a middle run at rank up to 64 (parity only)
]


@pytest.mark.parametrize("d,r,nrhs,dlevels,expect", DIAG_CASES)
def test_diagonal_levels(qtt, d, r, nrhs, dlevels, expect):
    """Cores with exact zeros off the (i, j) diagonal; where the planner picks
    the streaming "diag" stage it must; parity with the oracle, which knows
    nothing of the structure."""
    ranks, cores, x = random_case(3100 + d, d, r, nrhs)
    eye = np.eye(2).reshape(1, 2, 2, 1)
    for k in dlevels:
        cores[k] = np.ascontiguousarray(cores[k] * eye)
    y, st = gpu_apply(qtt, cores, x)
    oracle.assert_close(y, oracle.apply_alg2(cores, x))
    if expect:
        assert any(s["variant"] == "diag" for s in st), st


def test_diagonal_wide_outputs_kernel(qtt):
    """A diagonal run whose r_out exceeds 8 (lanes-over-outputs kernel): the
    bottom digits of a constant rank-24 profile, N = 2^18."""
    d, r = 18, 24
    ranks = [1] + [r] * (d - 1) + [1]
    _, cores, x = random_case(3300, d, r, 2, ranks=ranks)
    eye = np.eye(2).reshape(1, 2, 2, 1)
    for k in range(0, 6):
        cores[k] = np.ascontiguousarray(cores[k] * eye)
    y, st = gpu_apply(qtt, cores, x)
    oracle.assert_close(y, oracle.apply_alg2(cores, x))
    assert st[0]["variant"] == "diag" and st[0]["k_last"] == 6, st


def test_diagonal_stage_host_apply_bitwise(qtt):
    """qtt_apply_host with a diagonal last stage (chunked launches with row
    offsets): bitwise equal to the device apply."""
    from qtt_workload import bie_case
    _, M, _, _, x = bie_case(4, 16, 9, 12, 8, 1)
    with _per_stage(qtt, M) as op:
        assert op.stages()[-1]["variant"] == "diag", op.stages()
        yd = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        np.testing.assert_array_equal(op.apply_host(x), yd)


def test_diagonal_levels_planned(qtt):
    """The block-diagonal top digits become one diag stage (BIE factor M's shape)."""
    from qtt_workload import bie_case
    _, M, _, _, x = bie_case(2, 15, 6, 12, 8, 1)
    y, st = gpu_apply(qtt, M, x)
    diag = [s for s in st if s["variant"] == "diag"]
    assert diag and diag[-1]["k_last"] == 15 and diag[-1]["k_first"] <= 8, st
    oracle.assert_close(y, oracle.apply_alg2(M, x))


# ------------------------------------------------------------------ merged stages (super-cores)
@pytest.mark.parametrize("maxL", [1, 2, 3, 4, 6, 10])
@pytest.mark.parametrize("seed,d,maxr,nrhs", [(21, 10, 6, 3), (22, 13, 12, 2), (23, 15, 24, 1), (24, 9, 3, 7),
                                              (25, 14, 40, 2)])
def test_merged_stage_limits(qtt, maxL, seed, d, maxr, nrhs):
    """Every cap on the stage length gives the oracle's result (multi-RHS
    epilogue of merged stages included)."""
    ranks, cores, x = random_case(seed, d, maxr, nrhs)
    y, stages = gpu_apply(qtt, cores, x, max_stage_levels=maxL)
    assert all(s["k_last"] - s["k_first"] + 1 <= maxL for s in stages)
    oracle.assert_close(y, oracle.apply_alg2(cores, x))


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_config_plan_has_merged_stages(qtt, name):
    cfg, cores, _ = generate(name, with_x=False)
    op = _per_stage(qtt, cores)
    try:
        st = op.stages()
    finally:
        op.close()
    assert any(s["variant"] in ("merged", "wide") for s in st)
    assert st == qtt.plan_stages(cfg.ranks)


WIDE_CASES = [
    # ranks, nrhs: boundary stages whose super-core is streamed (variant "wide"),
    # odd r_out (scalar epilogue), r_out = 1, ragged M (< 64 rows), multi-RHS
    ([1, 2, 4, 8, 16, 32, 48, 48, 48, 32, 16, 8, 4, 2, 1], 1),
    ([1, 2, 4, 8, 16, 32, 48, 48, 48, 32, 16, 8, 4, 2, 1], 3),
    ([1, 2, 4, 8, 16, 24, 24, 24, 24, 24, 24, 24, 1], 2),
    ([1] + [20] * 11 + [1], 1),
    ([1] + [32] * 13 + [1], 2),
    ([1, 2, 4, 8, 16, 17, 17, 17, 9, 5, 3, 1], 5),
    ([1] + [40] * 9 + [1], 1),
]


@pytest.mark.parametrize("ranks,nrhs", WIDE_CASES)
def test_wide_stages(qtt, ranks, nrhs):
    d = len(ranks) - 1
    _, cores, x = random_case(300 + d + nrhs, d, max(ranks), nrhs, ranks=ranks)
    y, st = gpu_apply(qtt, cores, x)
    assert any(s["variant"] in ("wide", "small") for s in st), st
    oracle.assert_close(y, oracle.apply_alg2(cores, x))


_NO_SMALL_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1511_06029_b200 as q
import oracle
from qtt_workload import random_case
sys.path.insert(0, sys.argv[1] + "/tests")
from test_gpu_parity import WIDE_CASES
for ranks, nrhs in WIDE_CASES:
    d = len(ranks) - 1
    _, cores, x = random_case(300 + d + nrhs, d, max(ranks), nrhs, ranks=ranks)
    with q.QttOperator(cores, fused=False) as op:
        st = op.stages()
        assert any(s["variant"] == "wide" for s in st) and not any(s["variant"] == "small" for s in st), st
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    oracle.assert_close(y, oracle.apply_alg2(cores, x))
print("ok")
"""


def test_wide_stages_without_small_variant():
    """The same shapes with QTT_PLAN_NO_SMALL=1, so their boundary stages run on
    the wide (TMA, streamed super-core) kernel.  Subprocess: read once."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QTT_PLAN_NO_SMALL="1")
    r = subprocess.run([sys.executable, "-c", _NO_SMALL_SCRIPT, root], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_merged_closed_forms(qtt):
    """Merged stages on the exact closed forms: identity and shift stay bitwise."""
    d = 14
    x = np.random.default_rng(4).standard_normal((3, 1 << d))
    for maxL in (2, 5, 6, 10):
        y, st = gpu_apply(qtt, CF.identity_cores(d), x, max_stage_levels=maxL)
        assert any(s["k_last"] > s["k_first"] for s in st)       # multi-level stages
        np.testing.assert_array_equal(y, x)
        y, _ = gpu_apply(qtt, CF.shift_cores(d, 777), x, max_stage_levels=maxL)
        np.testing.assert_array_equal(y, np.roll(x, 777, axis=1))


# ------------------------------------------------------------------ BASELINE configs
@pytest.mark.parametrize("maxL", [1, None])
@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_config_full_vector(qtt, name, maxL):
    cfg, cores, x = generate(name)
    y, _ = gpu_apply(qtt, cores, x, max_stage_levels=maxL)
    ref = oracle.apply_alg2(cores, x)
    oracle.assert_close(y, ref)
    if name == "c1":
        oracle.assert_close(y, oracle.apply_dense(cores, x))


def test_c3x16_columns(qtt):
    cfg, cores, x = generate("c3x16")
    y, _ = gpu_apply(qtt, cores, x)
    # column 0 bitwise equal to the single-RHS run (deterministic, batch-invariant)
    _, cores1, x1 = generate("c3")
    y1, _ = gpu_apply(qtt, cores1, x1)
    np.testing.assert_array_equal(y[0], y1[0])
    for s in (0, 7, 15):
        oracle.assert_close(y[s:s + 1], oracle.apply_alg2(cores, x[s:s + 1]))


def _sampled_rows(N, n, seed):
    rng = np.random.default_rng(seed)
    rows = set(rng.integers(0, N, n).tolist()) | {0, 1, N // 2, N - 1}
    return np.array(sorted(rows))


@pytest.mark.parametrize("name,nrows", [("c4", 24)])
def test_full_size_sampled_rows(qtt, name, nrows):
    """Full BASELINE size, same launch configuration as bench.py; the oracle
    computes sampled outputs one by one (apply_rows: a third association of the
    sum, independent of the sweeps).  c5 is compared on every entry in
    test_gpu_full_parity.py (chunked oracle), which takes a fifth of the time
    10 sampled rows of c5 take here."""
    cfg, cores, x = generate(name)
    y, _ = gpu_apply(qtt, cores, x)
    assert np.all(np.isfinite(y))
    rows = _sampled_rows(cfg.N, nrows, 1)
    ref = oracle.apply_rows(cores, x, rows)
    rms = float(np.sqrt(np.mean(ref[0] ** 2)))
    oracle.assert_close(y[:, rows], ref, rms=rms, check_l2=False)
    m = oracle.compare(y[:, rows], ref, rms=rms)[0]
    assert m["rel_l2"] <= 1e-12, m


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_full_size_kronecker_vector(qtt, name):
    """x = v_d (x) ... (x) v_1: y = A x has exact TT cores from the compressed
    matvec; its entries are checked at sampled positions."""
    cfg, cores, _ = generate(name, with_x=False)
    rng = np.random.default_rng(5)
    vs = [rng.uniform(0.5, 1.5, 2) * rng.choice([-1, 1], 2) for _ in range(cfg.d)]
    xk = oracle.tt_vector_dense(oracle.kron_vector_cores(vs))[None, :]
    y, _ = gpu_apply(qtt, cores, xk)
    yc_cores = oracle.compressed_matvec(cores, oracle.kron_vector_cores(vs))
    rows = _sampled_rows(cfg.N, 2000, 2)
    ref = oracle.tt_vector_entries(yc_cores, rows)[None, :]
    rms = float(np.sqrt(np.mean(ref ** 2)))
    oracle.assert_close(y[:, rows], ref, rms=rms)


# ------------------------------------------------------------------ determinism, streams, ABI
def test_determinism_and_stream(qtt):
    _, cores, x = generate("c2")
    op = _per_stage(qtt, cores)
    xt = torch.from_numpy(x).cuda()
    y1 = op.apply(xt)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y2 = op.apply(xt, stream=s)
    s.synchronize()
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    # caller-owned workspace
    ws = torch.empty(op.workspace_size(1) // 8 + 32, dtype=torch.float64, device="cuda")
    y3 = op.apply(xt, workspace=ws)
    torch.cuda.synchronize()
    assert torch.equal(y1, y3)
    # host end-to-end entry point
    yh = op.apply_host(x)
    np.testing.assert_array_equal(yh, y1.cpu().numpy())
    op.close()


def test_abi_errors(qtt):
    lib = qtt._lib.load()
    import ctypes as C
    _, cores, x = generate("c1")
    op = _per_stage(qtt, cores)
    h = op.handle
    N = op.N
    xt = torch.from_numpy(x).cuda()
    big = torch.zeros(2 * N + 2, dtype=torch.float64, device="cuda")
    yt = torch.empty_like(xt)
    E = qtt._lib
    # nrhs < 1
    assert lib.qtt_apply(h, xt.data_ptr(), yt.data_ptr(), 0, None) == E.QTT_ERROR_INVALID_VALUE
    # overlap
    assert lib.qtt_apply(h, big.data_ptr(), big.data_ptr() + 8 * 8, 1, None) == E.QTT_ERROR_INVALID_VALUE
    # misaligned (8-byte offset)
    assert lib.qtt_apply(h, big.data_ptr() + 8, yt.data_ptr(), 1, None) == E.QTT_ERROR_NOT_SUPPORTED
    # host pointer
    assert lib.qtt_apply(h, x.ctypes.data, yt.data_ptr(), 1, None) == E.QTT_ERROR_NOT_SUPPORTED
    # null
    assert lib.qtt_apply(h, None, yt.data_ptr(), 1, None) == E.QTT_ERROR_INVALID_VALUE
    # a byte range beyond 2^63 (N * nrhs > 2^60) cannot be addressed
    too_many = (1 << 60) // N + 1
    assert lib.qtt_apply(h, xt.data_ptr(), yt.data_ptr(), too_many, None) == E.QTT_ERROR_INVALID_VALUE
    # short workspace
    ws = torch.empty(16, dtype=torch.float64, device="cuda")
    assert lib.qtt_apply_ws(h, xt.data_ptr(), yt.data_ptr(), 1, ws.data_ptr(), 128, None) == E.QTT_ERROR_INVALID_VALUE
    # python-side validation
    with pytest.raises(ValueError):
        op.apply(xt.float())
    with pytest.raises(ValueError):
        op.apply(torch.zeros(N + 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        op.apply(torch.zeros(N, dtype=torch.float64))
    # bad ranks at create
    with pytest.raises(qtt.QttError):
        qtt.qtt_create([np.zeros((2, 2, 2, 1))], ranks=[2, 1])
    op.close()
    assert lib.qtt_destroy(None) == E.QTT_SUCCESS


def test_apply_does_not_block_the_host(qtt):
    """qtt_apply only enqueues.  c4 takes ~55 ms on the device; the
    host call (graph replay after the first apply) returns in a small fraction."""
    import time
    cfg, cores, x = generate("c4")
    with _per_stage(qtt, cores) as op:
        xt = torch.from_numpy(x).cuda()
        y = torch.empty_like(xt)
        op.apply(xt, out=y)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        t0 = time.perf_counter()
        op.apply(xt, out=y)
        host_ms = (time.perf_counter() - t0) * 1e3
        b.record()
        b.synchronize()
        dev_ms = a.elapsed_time(b)
    assert dev_ms > 20.0 and host_ms < 0.1 * dev_ms, (host_ms, dev_ms)


def test_core_arrays_may_be_freed_after_create(qtt):
    """SURVEY T3 / qtt.h: qtt_create copies the cores; overwriting the caller's
    arrays afterwards does not change the operator."""
    _, cores, x = random_case(4321, 12, 9, 2)
    keep = [c.copy() for c in cores]
    op = _per_stage(qtt, cores)
    try:
        for c in cores:
            c.fill(np.nan)
        del cores
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    finally:
        op.close()
    oracle.assert_close(y, oracle.apply_alg2(keep, x))


def test_transpose_of(qtt):
    """QttOperator.transpose_of(cores) applies A^T: against the oracle on the
    pinned transpose (oracle.transpose), and <u, A v> = <A^T u, v>."""
    _, cores, x = random_case(4545, 12, 9, 2)
    with qtt.QttOperator.transpose_of(cores) as opT, _per_stage(qtt, cores) as op:
        xt = torch.from_numpy(x).cuda()
        yT = opT.apply(xt).cpu().numpy()
        y = op.apply(xt).cpu().numpy()
    oracle.assert_close(yT, oracle.apply_alg2(oracle.transpose(cores), x))
    u, v = x[0], x[1]
    lhs = float(u @ y[1])          # <u, A v>
    rhs = float(yT[0] @ v)         # <A^T u, v>
    assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs)), (lhs, rhs)


def test_operator_from_ttb1_file(qtt, tmp_path):
    """An operator loaded from a TTB1 core file applies bitwise like the same
    cores passed directly."""
    from paper_1511_06029_b200 import ttb1
    _, cores, x = generate("c2")
    ttb1.save(tmp_path / "c2.ttb1", cores)
    xt = torch.from_numpy(x).cuda()
    with qtt.QttOperator.from_ttb1(tmp_path / "c2.ttb1") as a, qtt.QttOperator(cores) as b:
        assert torch.equal(a.apply(xt), b.apply(xt))


def test_perf_regression_c4(qtt):
    """SURVEY T6 / BASELINE north_star: c4 must stay at >= 60% of the FP64
    roofline (Alg. 2 flops at the measured 37.08 TF/s DMMA peak); this build
    runs at ~105% on that basis (55.2 ms), so the bound only catches gross
    regressions.  Median of 5 applies, CUDA events."""
    cfg, cores, x = generate("c4")
    with _per_stage(qtt, cores) as op:
        xt = torch.from_numpy(x).cuda()
        y = torch.empty_like(xt)
        ts = []
        for i in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            op.apply(xt, out=y)
            b.record()
            b.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b))
        ms = sorted(ts)[len(ts) // 2]
        frac = op.flops_per_rhs / (ms * 1e-3) / 37.08e12
    assert frac >= 0.6, (ms, frac)
    assert ms < 70.0, ms


def test_nan_inf_propagate(qtt):
    d = 8
    _, cores, x = random_case(9, d, 6)
    x = x.copy()
    x[0, 5] = np.nan
    y, _ = gpu_apply(qtt, cores, x)
    ref = oracle.apply_alg2(cores, x)
    np.testing.assert_array_equal(np.isnan(y), np.isnan(ref))


def test_nan_stays_in_its_block_for_diagonal_levels(qtt):
    """DESIGN.md R21: diagonal cores are structural zeros -- a NaN in x reaches
    exactly the outputs of its own block (top digits equal), all others stay
    finite and match the oracle evaluated on the NaN-free blocks."""
    d, top = 12, 7
    ranks, cores, x = random_case(3100 + d, d, 6, 1)      # DIAG_CASES[0]: planned as a diag stage
    eye = np.eye(2).reshape(1, 2, 2, 1)
    for k in range(d - top, d):
        cores[k] = np.ascontiguousarray(cores[k] * eye)
    x = x.copy()
    j = 37
    x[0, j] = np.nan
    y, st = gpu_apply(qtt, cores, x)
    assert any(s["variant"] == "diag" for s in st), st
    blk = np.arange(1 << d) >> (d - top)
    inside = blk == (j >> (d - top))
    assert np.all(np.isnan(y[0, inside])) and np.all(np.isfinite(y[0, ~inside]))
    xz = x.copy()
    xz[0, j] = 0.0
    oracle.assert_close(y[:, ~inside], oracle.apply_alg2(cores, xz)[:, ~inside],
                        rms=float(np.sqrt(np.mean(oracle.apply_alg2(cores, xz) ** 2))), check_l2=False)


def test_caller_graph_capture(qtt):
    """The caller captures qtt_apply into its own CUDA graph (torch.cuda.graph):
    replays are bitwise equal to plain applies, plain applies on other streams
    still work afterwards (the captured event is not used for ordering), and a
    capture before the cached workspace exists is refused (NOT_SUPPORTED)."""
    _, cores, x = generate("c2")
    xt = torch.from_numpy(x).cuda()
    s = torch.cuda.Stream()
    with _per_stage(qtt, cores) as op:
        ref = op.apply(xt).clone()
        torch.cuda.synchronize()
        y = torch.empty_like(xt)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            op.apply(xt, out=y)
        for _ in range(3):
            y.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(y, ref)
        assert torch.equal(op.apply(xt), ref)
        del g
    with _per_stage(qtt, cores) as op:
        g = torch.cuda.CUDAGraph()
        y = torch.empty_like(xt)
        with pytest.raises(qtt.QttError):
            with torch.cuda.graph(g, stream=s):
                op.apply(xt, out=y)
        torch.cuda.synchronize()
        assert torch.equal(op.apply(xt), ref)


def test_graph_replay_matches_plain_enqueue(qtt):
    """Applies replay a cached CUDA graph per (x, y, workspace, nrhs); the result is
    bitwise that of the plain per-stage enqueue (stage timing on disables graphs),
    across alternating buffers, RHS counts and a non-default stream."""
    _, cores, x = random_case(31, 12, 9, 3)
    op = _per_stage(qtt, cores)
    try:
        xs = [torch.from_numpy(x).cuda(), torch.from_numpy(x[::-1].copy()).cuda(), torch.from_numpy(x[:1].copy()).cuda()]
        op.set_stage_timing(True)
        plain = [op.apply(t) for t in xs]
        torch.cuda.synchronize()
        op.stage_times()
        op.set_stage_timing(False)
        ys = [torch.empty_like(t) for t in xs]
        s = torch.cuda.Stream()
        for rep in range(3):
            for t, yb, p in zip(xs, ys, plain):
                yb.zero_()
                if rep == 2:
                    with torch.cuda.stream(s):
                        op.apply(t, out=yb, stream=s)
                    s.synchronize()
                else:
                    op.apply(t, out=yb)
                torch.cuda.synchronize()
                assert torch.equal(yb, p)
    finally:
        op.close()


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_apply_host_pipelined_bitwise(qtt, name):
    """qtt_apply_host overlaps the H2D of x with the first stage and the D2H of y
    with the last stage (chunked launches of the same kernels): bitwise equal
    to the device apply."""
    cfg, cores, x = generate(name)
    op = _per_stage(qtt, cores)
    try:
        yd = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        xh = torch.from_numpy(x).pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        for _ in range(2):
            yh.zero_()
            op.apply_host(xh.numpy(), out=yh.numpy())
            np.testing.assert_array_equal(yh.numpy(), yd)
        # pageable buffers too
        np.testing.assert_array_equal(op.apply_host(x), yd)
    finally:
        op.close()


_CHUNKED_HOST_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1511_06029_b200 as q
from qtt_workload import generate, random_case
cases = [("c3", None), ("split", (18, 64))]
for name, dr in cases:
    if dr is None:
        _, cores, x = generate(name)
    else:
        d, r = dr
        _, cores, x = random_case(6061, d, r, 1, ranks=[1] + [r] * (d - 1) + [1])
    with q.QttOperator(cores, fused=False) as op:
        yd = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        for _ in range(2):
            yh = op.apply_host(x)
            assert np.array_equal(yh, yd), name
print("ok")
"""


def test_apply_host_chunked_launches_bitwise():
    """QTT_NO_COPY_FLAGS=1 selects qtt_apply_host's other pipeline: the first
    and last stages run as 8 chunked launches each (split-K included, c3's and
    a constant-rank last stage); bitwise equal to the device apply.  Run in a
    subprocess because the switch is read once per process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QTT_NO_COPY_FLAGS="1")
    r = subprocess.run([sys.executable, "-c", _CHUNKED_HOST_SCRIPT, root], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


_FORCE_SMALL_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1511_06029_b200 as q
import oracle
from qtt_workload import random_case
cases = [(1, 1, 1, 1), (2, 2, 2, 5), (3, 3, 3, 7), (4, 6, 7, 3), (5, 9, 13, 2), (6, 10, 24, 1),
         (7, 12, 33, 1), (8, 13, 48, 2), (9, 14, 5, 4), (13, 11, 64, 1), (14, 9, 100, 1)]
n_small = 0
for seed, d, r, nrhs in cases:
    _, cores, x = random_case(seed + 900, d, r, nrhs)
    with q.QttOperator(cores, fused=False) as op:
        n_small += sum(s["variant"] == "small" for s in op.stages())
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    oracle.assert_close(y, oracle.apply_alg2(cores, x))
assert n_small > 20, n_small
print("ok", n_small)
"""


def test_small_variant_forced_everywhere():
    """QTT_PLAN_FORCE_SMALL=1 plans the warp-tile small kernel for every stage
    it can run (odd K, ragged rows and columns, multi-RHS); parity with the
    oracle.  Subprocess: the switch is read once per process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QTT_PLAN_FORCE_SMALL="1")
    r = subprocess.run([sys.executable, "-c", _FORCE_SMALL_SCRIPT, root], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("d,s,nrhs", [(28, 123457, 1), (26, 1, 3)])
def test_shift_large_d_bitwise(qtt, d, s, nrhs):
    """Large N (2 GiB vectors at d = 28; 64-bit offsets, many tiles): the exact
    rank-2 cyclic shift is np.roll / torch.roll bitwise."""
    gen = torch.Generator(device="cuda").manual_seed(d)
    x = torch.randn((nrhs, 1 << d), dtype=torch.float64, device="cuda", generator=gen)
    op = _per_stage(qtt, CF.shift_cores(d, s))
    try:
        y = op.apply(x)
        torch.cuda.synchronize()
        assert torch.equal(y, torch.roll(x, s, dims=1))
    finally:
        op.close()
    del x, y
    torch.cuda.empty_cache()


def test_back_to_back_applies_on_two_streams(qtt):
    """The cached workspace is shared: an apply enqueued on stream B right after
    one on stream A (no host sync between) is ordered after it by the library."""
    cfg, cores, x = generate("c3")
    x2 = np.ascontiguousarray(x[:, ::-1])
    op = _per_stage(qtt, cores)
    try:
        ref1 = op.apply(torch.from_numpy(x).cuda())
        ref2 = op.apply(torch.from_numpy(x2).cuda())
        torch.cuda.synchronize()
        a, b = torch.cuda.Stream(), torch.cuda.Stream()
        xa, xb = torch.from_numpy(x).cuda(), torch.from_numpy(x2).cuda()
        torch.cuda.synchronize()
        for _ in range(3):
            ya = op.apply(xa, stream=a)
            yb = op.apply(xb, stream=b)
            a.synchronize()
            b.synchronize()
            assert torch.equal(ya, ref1) and torch.equal(yb, ref2)
    finally:
        op.close()


def test_cached_ws_ordered_across_caller_ws_apply(qtt):
    """apply(A) on the cached workspace (stream a), apply_ws(B) with the
    caller's workspace (stream b), apply(C) on the cached workspace (stream c):
    C is ordered after A (the cached workspace's own event), not after B."""
    cfg, cores, x = generate("c3")
    xs = [x, np.ascontiguousarray(x[:, ::-1]), np.ascontiguousarray(-x)]
    op = _per_stage(qtt, cores)
    try:
        refs = [op.apply(torch.from_numpy(v).cuda()) for v in xs]
        torch.cuda.synchronize()
        ws = torch.empty(op.workspace_size(1) // 8 + 64, dtype=torch.float64, device="cuda")
        st = [torch.cuda.Stream() for _ in range(3)]
        xd = [torch.from_numpy(v).cuda() for v in xs]
        torch.cuda.synchronize()
        for _ in range(4):
            ya = op.apply(xd[0], stream=st[0])
            yb = torch.empty_like(xd[1])
            with torch.cuda.stream(st[1]):
                op.apply(xd[1], out=yb, workspace=ws, stream=st[1])
            yc = op.apply(xd[2], stream=st[2])
            for s_ in st:
                s_.synchronize()
            assert torch.equal(ya, refs[0]) and torch.equal(yb, refs[1]) and torch.equal(yc, refs[2])
    finally:
        op.close()


def test_cached_ws_grows_on_another_stream(qtt):
    """The cached workspace grows (nrhs 1 -> 4) on stream b while an apply that
    used the old block is still queued on stream a: the old block is released
    on b after a's apply (stream-ordered), and both results are right."""
    cfg, cores, x = generate("c3")
    x4 = np.ascontiguousarray(np.concatenate([x, -x, 2 * x, x[:, ::-1]]))
    op = _per_stage(qtt, cores)
    try:
        ref1 = op.apply(torch.from_numpy(x).cuda())
        ref4 = op.apply(torch.from_numpy(x4).cuda())
        torch.cuda.synchronize()
        for _ in range(2):
            op2 = _per_stage(qtt, cores)            # a fresh handle: workspace sized for nrhs = 1
            a, b = torch.cuda.Stream(), torch.cuda.Stream()
            xa, xb = torch.from_numpy(x).cuda(), torch.from_numpy(x4).cuda()
            torch.cuda.synchronize()
            ya = op2.apply(xa, stream=a)
            yb = op2.apply(xb, stream=b)
            a.synchronize()
            b.synchronize()
            assert torch.equal(ya, ref1) and torch.equal(yb, ref4)
            op2.close()
    finally:
        op.close()


def test_grid_apply_two_streams(qtt):
    """Grid applies on one handle from two streams share the staging vectors:
    the second is ordered after the first."""
    d = 15
    _, cores, _ = random_case(4242, d, 12)
    rng = np.random.default_rng(1)
    g1 = rng.standard_normal((1, 1 << d))
    g2 = rng.standard_normal((1, 1 << d))
    op = _per_stage(qtt, cores)
    try:
        r1 = op.apply_grid(torch.from_numpy(g1).cuda(), dim=3)
        r2 = op.apply_grid(torch.from_numpy(g2).cuda(), dim=3)
        torch.cuda.synchronize()
        a, b = torch.cuda.Stream(), torch.cuda.Stream()
        x1, x2 = torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda()
        torch.cuda.synchronize()
        for _ in range(3):
            y1 = op.apply_grid(x1, dim=3, stream=a)
            y2 = op.apply_grid(x2, dim=3, stream=b)
            a.synchronize()
            b.synchronize()
            assert torch.equal(y1, r1) and torch.equal(y2, r2)
    finally:
        op.close()


def test_apply_host_out_validation(qtt):
    _, cores, x = random_case(5, 8, 4, nrhs=2)
    op = _per_stage(qtt, cores)
    try:
        ref = op.apply_host(x)
        for bad in (np.empty(x.shape, dtype=np.float32), np.empty((x.shape[1],)),
                    np.empty((2, 2 * x.shape[1]))[:, ::2], np.empty((3, x.shape[1]))):
            with pytest.raises(ValueError):
                op.apply_host(x, out=bad)
        ro = np.empty_like(x)
        ro.flags.writeable = False
        with pytest.raises(ValueError):
            op.apply_host(x, out=ro)
        out = np.empty_like(x)
        assert op.apply_host(x, out=out) is out
        np.testing.assert_array_equal(out, ref)
    finally:
        op.close()


@pytest.mark.parametrize("seed", range(24))
def test_random_plan_fuzz(qtt, seed):
    """Random depth, rank profile (tapered, flat, spiky, odd) and RHS count
    through the default plan (whatever mix of resident / merged / wide /
    generic stages the scheduler picks) against the oracle."""
    rng = np.random.default_rng(9000 + seed)
    d = int(rng.integers(2, 17))
    kind = seed % 4
    if kind == 0:     # tapered like c4
        cap = int(rng.integers(2, 60))
        ranks = [min(2 ** k, 2 ** (d - k), cap) for k in range(d + 1)]
    elif kind == 1:   # flat
        r = int(rng.integers(1, 70))
        ranks = [1] + [r] * (d - 1) + [1]
    elif kind == 2:   # spiky
        ranks = [1] + [int(v) for v in rng.choice([1, 2, 3, 17, 40, 64, 96], d - 1)] + [1]
    else:             # uniform random
        ranks = [1] + [int(v) for v in rng.integers(1, 50, d - 1)] + [1]
    nrhs = int(rng.choice([1, 1, 2, 3, 5]))
    _, cores, x = random_case(9000 + seed, d, max(ranks), nrhs, ranks=ranks)
    y, st = gpu_apply(qtt, cores, x)
    oracle.assert_close(y, oracle.apply_alg2(cores, x))


def test_variant_fuzz_with_diagonal_runs(qtt):
    """80 random cases (d 1..18, ranks up to 64, nrhs 1..3, random stage caps),
    half with a random run of diagonal levels, against the oracle; together they
    exercise the merged, dmma, wide, small and diag kernels."""
    rng = np.random.default_rng(2025)
    seen = set()
    for c in range(80):
        d = int(rng.integers(1, 19))
        maxr = int(rng.choice([2, 5, 8, 16, 24, 33, 48, 64]))
        nrhs = int(rng.choice([1, 1, 2, 3]))
        ranks, cores, x = random_case(8000 + c, d, maxr, nrhs)
        if rng.random() < 0.5 and d >= 2:
            a = int(rng.integers(0, d))
            b = int(rng.integers(a, d)) + 1
            eye = np.eye(2).reshape(1, 2, 2, 1)
            for k in range(a, b):
                cores[k] = np.ascontiguousarray(cores[k] * eye)
        maxL = None if rng.random() < 0.6 else int(rng.integers(1, 11))
        y, st = gpu_apply(qtt, cores, x, max_stage_levels=maxL)
        seen.update(s["variant"] for s in st)
        oracle.assert_close(y, oracle.apply_alg2(cores, x))
    assert {"merged", "dmma", "wide", "small", "diag"} <= seen, seen


def test_graph_cache_eviction_and_workspace_growth(qtt):
    """More (x, y) pairs than the 8 cached graphs, and growing nrhs (the cached
    workspace is reallocated and graphs on the old one dropped): every result
    stays bitwise equal to the plain enqueue."""
    _, cores, x = random_case(41, 13, 20, 4)
    op = _per_stage(qtt, cores)
    try:
        xs = [torch.from_numpy(np.ascontiguousarray(np.roll(x, k, axis=1))).cuda() for k in range(11)]
        op.set_stage_timing(True)
        refs = [op.apply(t) for t in xs]
        torch.cuda.synchronize()
        op.stage_times()
        op.set_stage_timing(False)
        for rep in range(2):
            for t, ref in zip(xs, refs):
                assert torch.equal(op.apply(t), ref)
        # growing nrhs: 1 -> 4 -> 2 RHS through the cached workspace
        for n in (1, 4, 2):
            y = op.apply(xs[0][:n].contiguous())
            torch.cuda.synchronize()
            assert torch.equal(y, refs[0][:n])
    finally:
        op.close()


def test_plain_c_program_applies_the_shift(qtt, tmp_path):
    """examples/qtt_c_example.c: create / apply / destroy through include/qtt.h
    from plain C (no Python in the loop); the shift operator is exact, so the
    program checks y == roll(x, 1) bitwise."""
    import importlib.util
    import os
    import subprocess
    spec = importlib.util.spec_from_file_location(
        "abi_cpu", os.path.join(os.path.dirname(os.path.abspath(__file__)), "test_abi_cpu.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    exe, env = mod._build_c_example(tmp_path, qtt)
    r = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0 and " 0 of " in r.stdout, r.stdout + r.stderr
    assert "apply plan: 1 launch(es)" in r.stdout, r.stdout       # d = 12: the fused one-launch apply
