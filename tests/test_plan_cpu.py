"""Stage scheduler (host logic, no GPU): qtt_plan_stages through the C ABI.

A stage is a run of consecutive levels applied by one launch; L >= 2 levels
use the super-core (the QTT definition, PAPER Eq. TTdeccores P:519-523,
restricted to the stage's digits).  These tests check the schedule's
structure; its numerics are checked on the GPU (tests/test_gpu_parity.py).
"""
import pytest

from qtt_workload import configs


@pytest.fixture(scope="module")
def q():
    from paper_1511_06029_b200 import build
    build.build()
    import paper_1511_06029_b200 as q
    q._lib.load()
    return q


def check_cover(plan, d, max_levels):
    assert plan[0][0] == 1 and plan[-1][1] == d
    for (a0, b0, _), (a1, _, _) in zip(plan, plan[1:]):
        assert a1 == b0 + 1
    for a, b, v in plan:
        assert 1 <= b - a + 1 <= max_levels
        assert v in (0, 1, 2, 3, 4)
        if v == 2:
            assert b > a                    # merged: a super-core of several levels
        if v in (0, 1):
            assert b == a                   # generic / dmma: one level


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
@pytest.mark.parametrize("maxL", [1, 2, 3, 6, 10])
def test_plan_covers_levels(q, name, maxL):
    cfg = configs.make_config(name)
    plan = q.qtt_plan_stages(cfg.ranks, 0, maxL)
    check_cover(plan, cfg.d, maxL)
    if maxL == 1:
        assert len(plan) == cfg.d and all(v in (1, 3, 4) for _, _, v in plan)
        if cfg.N >= 1 << 21:
            assert all(v == 1 for _, _, v in plan)      # large N: smem-resident cores at r <= 48


def test_c4_plan_merges_tapered_ends_only(q):
    """c4 (r_k = min(2^k, 2^(24-k), 48)): the r=48 interior levels stay one per
    launch (a merge there would cost more flops or exceed the instance set);
    the tapered ends are merged, which removes HBM round trips and flops."""
    cfg = configs.make_config("c4")
    plan = q.qtt_plan_stages(cfg.ranks)
    for a, b, v in plan:
        if 8 <= a <= 17:
            assert a == b and v == 1
    assert plan[0][1] >= 2 and plan[-1][0] <= 23
    assert len(plan) < cfg.d


def test_small_problem_few_launches(q):
    # c1 (N = 4096) is latency-bound: the plan uses far fewer launches than levels
    cfg = configs.make_config("c1")
    assert len(q.qtt_plan_stages(cfg.ranks)) <= cfg.d // 2


def test_large_rank_levels_use_wide_kernel(q):
    # r = 70: 2 r = 140 > the smem-resident instances -> streamed super-core
    # ("wide"), or at tiny N the warp-tile "small" kernel; never generic
    ranks = [1, 2, 4] + [70] * 6 + [4, 2, 1]
    plan = q.qtt_plan_stages(ranks, 0, 1)
    assert all(v in (3, 4) for _, _, v in plan[2:9])
    assert all(v in (1, 3, 4) for _, _, v in plan)
    check_cover(q.qtt_plan_stages(ranks), len(ranks) - 1, 10)
    ranks = [1, 2, 4] + [70] * 11 + [4, 2, 1]                # N = 2^16: wide
    plan = q.qtt_plan_stages(ranks, 0, 1)
    assert [v for _, _, v in plan][2:13] == [3] * 11              # the r = 70 -> 70 levels


def test_huge_rank_falls_back_to_generic(q):
    # r_in = r_out = 1501: the level's super-core (3002 x 3002 doubles) exceeds 64 MiB
    plan = q.qtt_plan_stages([1, 2, 1501, 1501, 2, 1], 0, 1)
    assert [v for _, _, v in plan][2] == 0 and [v for _, _, v in plan][1] in (3, 4)


def test_split_k_only_for_few_tiles_and_long_k(q):
    """Split-K is planned only for wide stages whose output
    tiles leave SMs idle and whose work is large: the last stage of long
    constant-rank profiles.  Never for c4/c5 or the latency-bound c1/c2."""
    for name in ("c1", "c2", "c4", "c5"):
        assert all(s["ksplit"] == 1 for s in q.plan_stages(configs.make_config(name).ranks)), name
    c3 = q.plan_stages(configs.make_config("c3").ranks)
    assert [s["ksplit"] for s in c3][:-1] == [1] * (len(c3) - 1) and c3[-1]["ksplit"] > 1
    d, r = 18, 256
    plan = q.plan_stages([1] + [r] * (d - 1) + [1])
    last = plan[-1]
    assert last["variant"] == "wide" and last["k_last"] == d and last["ksplit"] > 1
    # every split is a non-empty k-range: S <= chunks, ceil(chunks / ceil(chunks / S)) == S
    L = last["k_last"] - last["k_first"] + 1
    chunks = -(-(2 ** L) * r // 32)
    S = last["ksplit"]
    cps = -(-chunks // S)
    assert -(-chunks // cps) == S
    # the split never changes which levels a stage covers
    check_cover([(s["k_first"], s["k_last"], 3 if s["variant"] == "wide" else 1 if s["variant"] == "dmma"
                  else 2 if s["variant"] == "merged" else 0) for s in plan], d, 10)


def test_small_variant_only_for_small_stages(q):
    """The warp-tile 'small' variant (no smem staging) is planned only where
    64-row TMA tiles cannot fill the GPU: never at N >= 2^21 (c3-c5)."""
    for name in ("c3", "c4", "c5"):
        assert all(s["variant"] != "small" for s in q.plan_stages(configs.make_config(name).ranks)), name
    assert q.plan_stages(configs.make_config("c1").ranks)[0]["variant"] == "small"


def test_rank_one_and_d1(q):
    assert q.qtt_plan_stages([1, 1]) == [(1, 1, 1)]
    plan = q.qtt_plan_stages([1] * 11)
    check_cover(plan, 10, 10)


def test_plan_validation(q):
    from paper_1511_06029_b200 import QttError
    with pytest.raises(QttError):
        q.qtt_plan_stages([2, 1])
    with pytest.raises(QttError):
        q.qtt_plan_stages([1, 0, 1])
    with pytest.raises(QttError):
        q.qtt_plan_stages([1, 2, 1], 0, 0)
    with pytest.raises(QttError):
        q.qtt_plan_stages([1] * 32)
    # the split variant validates the same way and accepts NULL outputs
    import ctypes as C
    lib = q._lib.load()
    n = C.c_int()
    r = (C.c_int64 * 3)(2, 1, 1)
    assert lib.qtt_plan_stages_split(2, r, 0, 10, C.byref(n), None, None, None, None) == q._lib.QTT_ERROR_INVALID_VALUE
    r = (C.c_int64 * 3)(1, 3, 1)
    assert lib.qtt_plan_stages_split(2, r, 0, 10, C.byref(n), None, None, None, None) == q._lib.QTT_SUCCESS
    assert n.value >= 1
    assert lib.qtt_plan_stages_split(2, r, 0, 10, None, None, None, None, None) == q._lib.QTT_ERROR_INVALID_VALUE


# --- super-cores (host logic of merged stages) --------------------------------
@pytest.mark.parametrize("ranks,k0,k1", [
    ([1, 3, 5, 2, 1], 1, 4),          # whole operator: W = dense A (r_0 = r_d = 1)
    ([1, 2, 4, 8, 16, 32, 6, 1], 1, 5),   # bottom stage, contracted left to right
    ([1, 6, 32, 16, 8, 4, 2, 1], 3, 7),   # top stage, contracted right to left
    ([1, 4, 7, 9, 3, 1], 2, 4),       # interior stage with open bonds at both ends
])
def test_super_core_is_the_qtt_definition(q, ranks, k0, k1):
    """W[a][ii][jj][b] from the library equals the product of core slices over
    the stage's digits (Eq. TTdeccores), i.e. the oracle's dense
    matrix of the sub-train with the open bonds fixed."""
    import numpy as np
    import oracle
    rng = np.random.default_rng(sum(ranks))
    d = len(ranks) - 1
    cores = [rng.standard_normal((ranks[k], 2, 2, ranks[k + 1])) for k in range(d)]
    W = q.stage_super_core(cores, k0, k1)
    sub = cores[k0 - 1:k1]
    L = k1 - k0 + 1
    assert W.shape == (ranks[k0 - 1], 1 << L, 1 << L, ranks[k1])
    for a in range(ranks[k0 - 1]):
        for b in range(ranks[k1]):
            # close the open bonds with unit vectors -> an ordinary QTT (r = 1 ends)
            first = sub[0][a:a + 1]
            last = sub[-1][..., b:b + 1]
            closed = [first] + sub[1:-1] + [last] if L > 1 else [sub[0][a:a + 1, :, :, b:b + 1]]
            np.testing.assert_allclose(W[a, :, :, b], oracle.dense_matrix(closed), rtol=1e-12, atol=1e-12)


def test_forced_stage_split_switch():
    """QTT_PLAN_FORCE_STAGES (A/B diagnostic, read once per process) forces the
    partition when it covers 1..d with coverable stages, and is ignored
    otherwise (the default plan stays)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, sys.argv[1]); import paper_1511_06029_b200 as q; "
            "from qtt_workload import configs; r = configs.config_ranks('c4'); "
            "print([(a, b) for a, b, _ in q.qtt_plan_stages(r, 0, 10)])")
    def run(spec):
        env = dict(os.environ)
        if spec is not None:
            env["QTT_PLAN_FORCE_STAGES"] = spec
        r = subprocess.run([sys.executable, "-c", code, root], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        return eval(r.stdout.strip().splitlines()[-1])
    default = run(None)
    pairs = "1-7,8-9,10-11,12-13,14-15,16-17,18-24"
    assert run(pairs) == [(1, 7), (8, 9), (10, 11), (12, 13), (14, 15), (16, 17), (18, 24)]
    singles = "1-7," + ",".join(str(k) for k in range(8, 18)) + ",18-24"   # "k" = the stage k-k
    assert run(singles) == [(1, 7)] + [(k, k) for k in range(8, 18)] + [(18, 24)]
    assert run("1-7,8-9") == default            # does not reach d = 24
    assert run("2-24") == default               # does not start at level 1
    assert run("garbage") == default


def test_fused_unit_division_magic():
    """The fused kernel divides a work-unit index u < 2^31 by its row-group
    count with a multiply and a shift (qtt_runtime.cpp enqueue_fused,
    qtt_wide_kernel.cu fused_cb): a power of two is a shift, otherwise
    mul = floor(2^(31+l) / d) + 1 with l = ceil(log2 d) and
    u / d = umulhi(u, mul) >> (l - 1).  Checked here against integer division
    for every divisor up to 4096 on the units a kernel can see, and on
    random indices up to 2^31 - 1."""
    import random
    rng = random.Random(0)
    for d in range(1, 4097):
        l = 0
        while (1 << l) < d:
            l += 1
        if d & (d - 1) == 0:
            div = lambda u: u >> l
        else:
            mul = ((1 << (31 + l)) // d) + 1
            assert mul < (1 << 32)
            div = lambda u: ((u * mul) >> 32) >> (l - 1)
        us = list(range(0, 4 * d + 3)) + [rng.randrange(0, 1 << 31) for _ in range(64)] + [(1 << 31) - 1]
        for u in us:
            assert div(u) == u // d, (d, u)
