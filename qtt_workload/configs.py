"""The five BASELINE.json configurations (c1..c5, c3 also with 16 RHS).

Each config stands in for a row of the paper's volume-integral experiments
(Tables 1-2): the paper's inverse cores
come from DMRG/AMEN inversion of a Laplace volume operator, which is out of
scope, so random cores with the stated rank profile stand in for them.  The
apply's cost depends only on the rank profile.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    d: int
    ranks: tuple            # r_0..r_d
    core_scale: tuple       # per-core scale factor applied to N(0,1) draws
    x_dist: str             # "normal" or "uniform"
    nrhs: int
    seed: int
    stands_for: str

    @property
    def N(self) -> int:
        return 1 << self.d


def config_ranks(name: str) -> List[int]:
    return list(make_config(name).ranks)


def _const_ranks(d: int, r: int) -> tuple:
    return tuple([1] + [r] * (d - 1) + [1])


def make_config(name: str, seed: int = 0) -> Config:
    """BASELINE.json configs; seed 0 for all."""
    if name == "c1":
        d, r = 12, 8
        ranks = _const_ranks(d, r)
        return Config(name, d, ranks, tuple([1 / math.sqrt(2 * r)] * d), "normal", 1, seed,
                      "1-D quantized, N=4096 (Tables 1-2 row 16^3 size)")
    if name == "c2":
        d, r = 15, 16
        ranks = _const_ranks(d, r)
        return Config(name, d, ranks, tuple([1 / math.sqrt(2 * r)] * d), "normal", 1, seed,
                      "3-D volume 32^3 (Tables 1-2 row 32^3)")
    if name in ("c3", "c3x16"):
        d, r = 21, 32
        ranks = _const_ranks(d, r)
        return Config(name, d, ranks, tuple([1 / math.sqrt(2 * r)] * d), "normal",
                      16 if name == "c3x16" else 1, seed,
                      "3-D volume 128^3 (Tables 1-2 row 128^3; GMRES preconditioner apply)")
    if name == "c4":
        d = 24
        ranks = tuple(min(2 ** k, 2 ** (d - k), 48) for k in range(d + 1))
        scale = tuple(1 / math.sqrt(2 * ranks[k]) for k in range(d))  # 1/sqrt(2 r_{k-1})
        return Config(name, d, ranks, scale, "uniform", 1, seed,
                      "3-D volume 256^3 (Tables 1-2 row 256^3, inverse max rank 57/62)")
    if name == "c5":
        d, r = 27, 24
        ranks = _const_ranks(d, r)
        return Config(name, d, ranks, tuple([1 / math.sqrt(2 * r)] * d), "normal", 1, seed,
                      "3-D volume 512^3 (beyond the paper, N ~ 1e8 per P:189-192)")
    raise KeyError(name)


CONFIGS = ("c1", "c2", "c3", "c3x16", "c4", "c5")


def flops_per_apply(ranks, nrhs: int = 1) -> int:
    """Algorithmic flops of one apply: 4 * sum_k r_{k-1} r_k * N * nrhs.

    PAPER.md P:1525-1528 counts 2 m_k r_{k+1} r_k N "operations" per level
    (with the off-by-one garble resolved as in SURVEY R3/R4); with m_k = 2 and
    one multiply-add counted as two flops this is 4 r_{k-1} r_k N.
    """
    d = len(ranks) - 1
    s = sum(int(ranks[k]) * int(ranks[k + 1]) for k in range(d))
    return 4 * s * (1 << d) * nrhs
