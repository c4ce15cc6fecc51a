"""Oracle for the Morton (hierarchical) ordering of grid samples -- TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:1625-1628: the N = 2^d grid points are indexed "according to
successive bisection of the domain along each coordinate direction (i.e.,
Morton ordered)"; Remark rem:interlace.  Convention (DESIGN.md
R18): QTT-order index q has bit ``dim*l + a`` equal to bit ``l``
of coordinate ``a`` (a = 0 x, 1 y, 2 z; l = 0 the finest level); the natural
grid is C-order ``[z][y][x]`` (x fastest).  Plain loops over bits.
"""
from __future__ import annotations

import numpy as np


def morton_coords(q: int, dim: int, levels: int):
    """Coordinates (x, y, z)[:dim] of QTT-order index q (loop over bits)."""
    c = [0] * dim
    for l in range(levels):
        for a in range(dim):
            c[a] |= ((q >> (dim * l + a)) & 1) << l
    return tuple(c)


def natural_index(c, levels: int) -> int:
    """C-order offset of coordinates c = (x, y, z)[:dim] in an n^dim grid, n = 2^levels."""
    off = 0
    for a in reversed(range(len(c))):
        off = (off << levels) | c[a]
    return off


def morton_perm(dim: int, levels: int) -> np.ndarray:
    """p with x_qtt[q] = grid_flat[p[q]] (q = 0..N-1)."""
    N = 1 << (dim * levels)
    return np.array([natural_index(morton_coords(q, dim, levels), levels) for q in range(N)], dtype=np.int64)


def pack(grid: np.ndarray, dim: int, levels: int) -> np.ndarray:
    """grid (nrhs, n^dim natural order) -> (nrhs, N) QTT order."""
    g = np.atleast_2d(grid)
    return g[:, morton_perm(dim, levels)]


def unpack(x: np.ndarray, dim: int, levels: int) -> np.ndarray:
    """(nrhs, N) QTT order -> natural grid order (inverse of pack)."""
    x = np.atleast_2d(x)
    out = np.empty_like(x)
    out[:, morton_perm(dim, levels)] = x
    return out
