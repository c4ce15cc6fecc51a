"""Seeded draws of QTT cores and dense right-hand sides.

Draw order: one ``numpy.random.Generator(PCG64(seed))`` per
config; cores first, k = 1..d, each ``standard_normal((r_{k-1},2,2,r_k))`` in
C order then scaled; then x as ``standard_normal((nrhs, N))`` (c4:
``uniform(-1, 1, (1, N))``).  Hence c3x16's first RHS equals c3's x.
"""
from __future__ import annotations

import numpy as np

from .configs import make_config


def random_cores(rng: np.random.Generator, ranks, scale=None):
    d = len(ranks) - 1
    cores = []
    for k in range(d):
        g = rng.standard_normal((ranks[k], 2, 2, ranks[k + 1]))
        if scale is not None:
            s = scale[k] if np.ndim(scale) else scale
            g *= s
        cores.append(np.ascontiguousarray(g, dtype=np.float64))
    return cores


def generate(name: str, seed: int = 0, with_x: bool = True):
    """Return (cfg, cores, x) for a BASELINE config; x has shape (nrhs, N)."""
    cfg = make_config(name, seed)
    rng = np.random.Generator(np.random.PCG64(seed))
    cores = random_cores(rng, cfg.ranks, cfg.core_scale)
    x = None
    if with_x:
        if cfg.x_dist == "uniform":
            x = rng.uniform(-1.0, 1.0, (cfg.nrhs, cfg.N))
        else:
            x = rng.standard_normal((cfg.nrhs, cfg.N))
    return cfg, cores, x


def rank_profile_random(rng: np.random.Generator, d: int, max_rank: int):
    """A random valid rank profile r_0 = r_d = 1, 1 <= r_k <= max_rank."""
    inner = rng.integers(1, max_rank + 1, size=max(d - 1, 0)).tolist()
    return [1] + inner + [1]


def random_case(seed: int, d: int, max_rank: int, nrhs: int = 1, ranks=None):
    """Random cores (scaled 1/sqrt(2 r_{k-1})) and x ~ N(0,1) for parity sweeps."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if ranks is None:
        ranks = rank_profile_random(rng, d, max_rank)
    scale = [1.0 / np.sqrt(2.0 * ranks[k]) for k in range(d)]
    cores = random_cores(rng, ranks, scale)
    x = rng.standard_normal((nrhs, 1 << d))
    return list(ranks), cores, x


def random_tt_vector(seed: int, d: int, max_rank: int, ranks=None):
    """A random TT vector (cores (r_{k-1}, 2, r_k), scaled 1/sqrt(2 r_{k-1})) for the
    compressed matvec (PAPER section 4.2); returns (ranks, cores)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if ranks is None:
        ranks = rank_profile_random(rng, d, max_rank)
    cores = []
    for k in range(d):
        g = rng.standard_normal((ranks[k], 2, ranks[k + 1])) / np.sqrt(2.0 * ranks[k])
        cores.append(np.ascontiguousarray(g))
    return list(ranks), cores


def bie_case(seed: int = 0, d: int = 21, point_bits: int = 9, r_y: int = 95, r_m: int = 50, nrhs: int = 1):
    """Synthetic stand-in for the paper's boundary-integral preconditioner
    (Table 3; product form X = M Y): N = 2^d
    unknowns = 2^(d - point_bits) surfaces x 2^point_bits points per surface
    (the paper's largest case, 4096 surfaces x 480 points = 1,966,080, padded
    to 512 points: d = 21).  Y: dense cores with tapered ranks
    min(2^k, 2^(d-k), r_y) (inverse max rank 95 in Table 3).  M: block-diagonal
    over surfaces -- cores of the surface digits k > point_bits are diagonal in
    (i_k, j_k) -- with ranks min(2^k, 2^(d-k), r_m) (the parenthesised 50).
    Scales 1/sqrt(2 r_{k-1}).  Returns (ranks_M, cores_M, ranks_Y, cores_Y, x);
    x ~ N(0,1) of shape (nrhs, N).  Apply as QttProduct([M, Y])."""
    rng = np.random.Generator(np.random.PCG64(seed))
    ranks_y = [min(2 ** k, 2 ** (d - k), r_y) for k in range(d + 1)]
    ranks_m = [min(2 ** k, 2 ** (d - k), r_m) for k in range(d + 1)]
    cores_y = random_cores(rng, ranks_y, [1.0 / np.sqrt(2.0 * ranks_y[k]) for k in range(d)])
    cores_m = random_cores(rng, ranks_m, [1.0 / np.sqrt(2.0 * ranks_m[k]) for k in range(d)])
    diag = np.eye(2).reshape(1, 2, 2, 1)
    for k in range(point_bits, d):          # 0-based core k acts on digit k+1: the surface digits
        cores_m[k] = np.ascontiguousarray(cores_m[k] * diag)
    x = rng.standard_normal((nrhs, 1 << d))
    return ranks_m, cores_m, ranks_y, cores_y, x
