"""The fused apply (variant 'fused'): every stage of a
latency-bound apply in ONE persistent launch, grid barriers between stages.

Parity against the CPU oracle (Alg. 2) and the closed forms, on
the default plans of c1 / c2 (where the cost model picks it), on random
profiles with d <= 15 forced through it (QTT_FORCE_FUSED=1, subprocess: the
switch is read once per process), through both entry points (cached
workspace, caller workspace), across RHS counts, and bitwise against the
per-stage launches of the same handle (stage timing runs those).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from qtt_workload import closed_forms as CF
from qtt_workload import generate, random_case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def qtt():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    import paper_1511_06029_b200 as q
    q._lib.load()
    return q


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_default_plan_is_one_launch(qtt, name):
    cfg, cores, x = generate(name)
    with qtt.QttOperator(cores) as op:
        assert op.launches(1) == 1
        st = op.stages(1)
        assert st and all(s["variant"] == "fused" for s in st)
        assert st[0]["k_first"] == 1 and st[-1]["k_last"] == cfg.d
        assert all(a["k_last"] + 1 == b["k_first"] for a, b in zip(st, st[1:]))
        y = op.apply(torch.from_numpy(x).cuda())
        # the per-stage launches of the same handle (stage timing runs those)
        op.set_stage_timing(True)
        assert op.launches(1) > 1
        y2 = op.apply(torch.from_numpy(x).cuda())
        op.set_stage_timing(False)
        op.stage_times()
        torch.cuda.synchronize()
        y, y2 = y.cpu().numpy(), y2.cpu().numpy()
    ref = oracle.apply_blas_sweep(cores, x)
    oracle.assert_close(y, ref)
    oracle.assert_close(y2, ref)
    if name == "c1":
        oracle.assert_close(y, oracle.apply_dense(cores, x))


def test_fused_entry_points_and_repeats(qtt):
    """Cached workspace (barrier words kept at 0 between launches) and caller
    workspace (cleared per apply); 50 back-to-back applies with alternating
    inputs, bitwise reproducible."""
    cfg, cores, x = generate("c2")
    x2 = np.ascontiguousarray(x[:, ::-1])
    with qtt.QttOperator(cores) as op:
        assert op.launches(1) == 1
        xa, xb = torch.from_numpy(x).cuda(), torch.from_numpy(x2).cuda()
        ra, rb = op.apply(xa), op.apply(xb)
        ws = torch.empty(op.workspace_size(1) // 8 + 64, dtype=torch.float64, device="cuda")
        ws.fill_(np.nan)                       # garbage in the caller's workspace
        ya, yb = torch.empty_like(xa), torch.empty_like(xb)
        for i in range(50):
            if i % 2:
                op.apply(xa, out=ya)
                op.apply(xb, out=yb, workspace=ws)
            else:
                op.apply(xb, out=yb)
                op.apply(xa, out=ya, workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(ya, ra) and torch.equal(yb, rb)
    oracle.assert_close(ra.cpu().numpy(), oracle.apply_blas_sweep(cores, x))


@pytest.mark.parametrize("nrhs", [2, 3, 4])
def test_fused_multi_rhs(qtt, nrhs):
    cfg, cores, _ = generate("c1")
    x = np.random.default_rng(nrhs).standard_normal((nrhs, cfg.N))
    with qtt.QttOperator(cores) as op:
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        y1 = op.apply(torch.from_numpy(np.ascontiguousarray(x[:1])).cuda()).cpu().numpy()
        both_fused = op.launches(nrhs) == 1 and op.launches(1) == 1
    oracle.assert_close(y, oracle.apply_blas_sweep(cores, x))
    if both_fused:
        np.testing.assert_array_equal(y[0], y1[0])      # the same stage split: batch-invariant


def test_fused_closed_forms(qtt):
    """Exact closed forms through the fused launch: identity and the cyclic
    shift, bitwise."""
    d = 13
    x = np.random.default_rng(0).standard_normal((2, 1 << d))
    for cores, ref in ((CF.identity_cores(d), x), (CF.shift_cores(d, 777), np.roll(x, 777, axis=1))):
        with qtt.QttOperator(cores) as op:
            y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        np.testing.assert_array_equal(y, ref)


_FORCE_FUSED_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1511_06029_b200 as q
import oracle
from qtt_workload import random_case
from qtt_workload import closed_forms as CF
cases = [(1, 1, 1, 1), (2, 2, 2, 5), (3, 3, 3, 7), (4, 6, 7, 3), (5, 9, 13, 2), (6, 10, 24, 1),
         (7, 12, 33, 1), (8, 13, 48, 2), (9, 14, 5, 4), (10, 15, 16, 1), (13, 11, 64, 1), (14, 9, 100, 1),
         (15, 15, 31, 1), (16, 8, 3, 16)]
n_fused = 0
for seed, d, r, nrhs in cases:
    _, cores, x = random_case(seed + 1900, d, r, nrhs)
    with q.QttOperator(cores) as op:
        fused = op.launches(nrhs) == 1 and op.stages(nrhs)[0]["variant"] == "fused"
        n_fused += fused
        xt = torch.from_numpy(x).cuda()
        y = op.apply(xt).cpu().numpy()
        ws = torch.empty(op.workspace_size(nrhs) // 8 + 64, dtype=torch.float64, device="cuda")
        yw = op.apply(xt, workspace=ws).cpu().numpy()
    oracle.assert_close(y, oracle.apply_alg2(cores, x))
    assert np.array_equal(y, yw), (seed, d, r)
for d in (4, 11, 15):
    x = np.random.default_rng(d).standard_normal((1, 1 << d))
    with q.QttOperator(CF.shift_cores(d, 5)) as op:
        assert op.launches(1) == 1
        assert np.array_equal(op.apply(torch.from_numpy(x).cuda()).cpu().numpy(), np.roll(x, 5, axis=1))
assert n_fused >= 12, n_fused
print("ok", n_fused)
"""


def test_fused_forced_random_profiles():
    env = dict(os.environ, QTT_FORCE_FUSED="1")
    r = subprocess.run([sys.executable, "-c", _FORCE_FUSED_SCRIPT, ROOT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_fused_disabled_switch():
    code = ("import sys; sys.path.insert(0, sys.argv[1]); import paper_1511_06029_b200 as q; "
            "from qtt_workload import generate; cfg, cores, x = generate('c1'); op = q.QttOperator(cores); "
            "print('launches', op.launches(1), op.stages(1)[0]['variant'])")
    r = subprocess.run([sys.executable, "-c", code, ROOT], env=dict(os.environ, QTT_NO_FUSED="1"),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "fused" not in r.stdout and "launches 1 " not in r.stdout, r.stdout


@pytest.mark.parametrize("name,dim,nrhs", [("c1", 3, 1), ("c1", 2, 1), ("c1", 3, 2), ("c2", 3, 1), ("c2", 1, 1)])
def test_fused_grid_apply_morton(qtt, name, dim, nrhs):
    """qtt_apply_grid on a fused plan: the Morton gather / scatter run inside
    the first / last stage of the one launch (no staging vectors); against the
    oracle's Morton pack (R18) + Alg. 2 + unpack, and bitwise
    against the staged path (QttOperator with the per-stage plan: stage timing on)."""
    from oracle import morton as OM
    cfg, cores, _ = generate(name)
    if cfg.d % dim:
        pytest.skip("dim must divide d")
    levels = cfg.d // dim
    g = np.random.default_rng(7 + dim).standard_normal((nrhs, cfg.N))
    with qtt.QttOperator(cores) as op:
        assert op.launches(nrhs) == 1
        y = op.apply_grid(torch.from_numpy(g).cuda(), dim).cpu().numpy()
        # the same operator's per-stage path (pack, stages, unpack)
        op.set_stage_timing(True)
        y2 = op.apply_grid(torch.from_numpy(g).cuda(), dim).cpu().numpy()
        op.set_stage_timing(False)
        op.stage_times()
    ref = OM.unpack(oracle.apply_blas_sweep(cores, OM.pack(g, dim, levels)), dim, levels)
    oracle.assert_close(y, ref)
    oracle.assert_close(y2, ref)


def test_fused_grid_apply_shift_bitwise(qtt):
    """The exact cyclic shift through a fused grid apply: natural order in,
    natural order out, bitwise (y = unpack(roll(pack(g))))."""
    from oracle import morton as OM
    d, dim = 12, 3
    g = np.random.default_rng(3).standard_normal((1, 1 << d))
    with qtt.QttOperator(CF.shift_cores(d, 9)) as op:
        assert op.launches(1) == 1
        y = op.apply_grid(torch.from_numpy(g).cuda(), dim).cpu().numpy()
    ref = OM.unpack(np.roll(OM.pack(g, dim, d // dim), 9, axis=1), dim, d // dim)
    np.testing.assert_array_equal(y, ref)


def test_fused_caller_graph_capture(qtt):
    """The caller captures a fused apply (one cooperative launch, no memset on
    the handle's own workspace) into a CUDA graph: replays are bitwise the
    plain apply, and plain applies still work afterwards."""
    _, cores, x = generate("c1")
    xt = torch.from_numpy(x).cuda()
    s = torch.cuda.Stream()
    with qtt.QttOperator(cores) as op:
        assert op.launches(1) == 1
        ref = op.apply(xt).clone()
        torch.cuda.synchronize()
        y = torch.empty_like(xt)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            op.apply(xt, out=y)
        for _ in range(5):
            y.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(y, ref)
        assert torch.equal(op.apply(xt), ref)
        del g


def test_stage_cap_disables_fused(qtt):
    """A caller-capped stage length (qtt_create_ex, e.g. 1 = Alg. 2 level by
    level) asks for that launch structure: no fused plan is built."""
    cfg, cores, x = generate("c1")
    with qtt.QttOperator(cores, max_stage_levels=1) as op:
        assert op.launches(1) == cfg.d
        assert all(s["variant"] != "fused" for s in op.stages(1))
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    oracle.assert_close(y, oracle.apply_dense(cores, x))


_MODES_SCRIPT = r"""
import hashlib, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1511_06029_b200 as q
from qtt_workload import generate, random_case
h = hashlib.sha256()
runs = []
for name in ("c1", "c2"):
    cfg, cores, x = generate(name)
    runs.append((cores, x))
for seed, d, r, nrhs in ((3, 12, 8, 2), (5, 13, 16, 1), (8, 14, 12, 3), (11, 10, 32, 1)):
    _, cores, x = random_case(seed + 2100, d, r, nrhs)
    runs.append((cores, x))
n_fused = 0
for cores, x in runs:
    with q.QttOperator(cores) as op:
        n_fused += op.stages(x.shape[0])[0]["variant"] == "fused"
        xt = torch.from_numpy(x).cuda()
        ws = torch.empty(op.workspace_size(x.shape[0]) // 8 + 64, dtype=torch.float64, device="cuda")
        for _ in range(3):   # cached workspace (first apply clears it, later ones replay), caller workspace
            h.update(op.apply(xt).cpu().numpy().tobytes())
            h.update(op.apply(xt, workspace=ws).cpu().numpy().tobytes())
print("digest", h.hexdigest(), n_fused)
"""


def test_fused_launch_modes_bitwise():
    """The fused apply's launch modes give bitwise-identical results: the
    default non-cooperative PDL launch, the cooperative launch replayed from a
    cached graph (QTT_FUSED_COOP=1), and the scattered per-warp epilogue
    (QTT_FUSED_NO_RUNS=1) against the run-wise smem epilogue whose split-K
    reduction keeps the summation order 0..ks-1."""
    out = {}
    for tag, extra in (("default", {}), ("coop", {"QTT_FUSED_COOP": "1"}), ("noruns", {"QTT_FUSED_NO_RUNS": "1"}),
                       ("forced", {"QTT_FORCE_FUSED": "1"})):
        r = subprocess.run([sys.executable, "-c", _MODES_SCRIPT, ROOT], env=dict(os.environ, **extra),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and "digest" in r.stdout, tag + ": " + r.stdout + r.stderr
        dig, nf = r.stdout.split("digest")[1].split()
        out[tag] = (dig, int(nf))
    assert out["default"][1] >= 2 and out["forced"][1] >= 5, out
    assert out["default"][0] == out["coop"][0] == out["noruns"][0], out


def test_fused_concurrent_with_other_kernels(qtt):
    """The fused launch is not cooperative: its CTAs may
    become resident at different times when other kernels hold SMs.  Run
    fused applies on one stream while large GEMMs run on another stream of
    the same device; every result must equal the isolated apply bitwise (and
    the barrier must not hang)."""
    _, cores, x = generate("c2")
    xt = torch.from_numpy(x).cuda()
    a = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with qtt.QttOperator(cores) as op:
        assert op.stages(1)[0]["variant"] == "fused"
        ref = op.apply(xt).clone()
        torch.cuda.synchronize()
        outs = [torch.empty_like(xt) for _ in range(40)]
        with torch.cuda.stream(s2):
            c = a
            for _ in range(6):
                c = torch.mm(c, a) * 1e-3
        for y in outs:
            op.apply(xt, out=y, stream=s1)
        torch.cuda.synchronize()
    for y in outs:
        assert torch.equal(y, ref)


_GRID_SCRIPT = r"""
import hashlib, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1511_06029_b200 as q
from qtt_workload import generate
h = hashlib.sha256()
for name, dim, nrhs in (("c1", 3, 1), ("c1", 2, 2), ("c1", 1, 1)):
    cfg, cores, _ = generate(name)
    x = np.random.default_rng(nrhs + dim).standard_normal((nrhs, cfg.N))
    with q.QttOperator(cores) as op:
        g = op.apply_grid(torch.from_numpy(x).cuda(), dim)
        h.update(g.cpu().numpy().tobytes())
print("digest", h.hexdigest())
"""


def test_fused_grid_gather_modes_bitwise():
    """Fused grid apply: the Morton gather inside stage 0's A loads (default
    for small grids) and the gather pre-pass + grid barrier
    (QTT_FUSED_PREPASS=1) give bitwise-identical results."""
    out = []
    for extra in ({}, {"QTT_FUSED_PREPASS": "1"}):
        r = subprocess.run([sys.executable, "-c", _GRID_SCRIPT, ROOT], env=dict(os.environ, **extra),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and "digest" in r.stdout, r.stdout + r.stderr
        out.append(r.stdout.split("digest")[1].strip())
    assert out[0] == out[1]


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_fused_apply_host_same_bits(qtt, name):
    """qtt_apply_host on a handle whose applies are fused runs the same plan
    (H2D, the fused launch, D2H), so its result is bitwise that of qtt_apply."""
    _, cores, x = generate(name)
    with qtt.QttOperator(cores) as op:
        assert op.stages(1)[0]["variant"] == "fused"
        yd = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        xh = torch.from_numpy(x).pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        for _ in range(3):
            yh.zero_()
            op.apply_host(xh.numpy(), out=yh.numpy())
            np.testing.assert_array_equal(yh.numpy(), yd)
        np.testing.assert_array_equal(op.apply_host(x), yd)
