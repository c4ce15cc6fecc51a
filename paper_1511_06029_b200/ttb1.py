"""TTB1 core files: load QTT operators written by other tools.

Layout (little-endian): magic b"TTB1"; u32 d; u32 flag (0 vector, 1 operator);
d x u32 row mode sizes; d x u32 column mode sizes (all 1 for vectors);
(d + 1) x u32 ranks; then the cores in order, each r_{k-1} x (m_k n_k) x r_k
float64 in row-major order (alpha_{k-1} slowest, alpha_k fastest; the pair
(i_k, j_k) flattened with the row digit i_k major -- DESIGN.md reading R2).
Readers reject anything whose payload does not match the header.

Host-side file I/O only (plumbing): the cores go to ``QttOperator`` as usual.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"TTB1"


def save(path, cores, vector: bool = False) -> None:
    """Write operator cores (r, 2, 2, r') -- or vector cores (r, 2, r') with vector=True."""
    d = len(cores)
    arrs = [np.ascontiguousarray(np.asarray(c, dtype="<f8")) for c in cores]
    if vector:
        rows = [a.shape[1] for a in arrs]
        cols = [1] * d
    else:
        rows = [a.shape[1] for a in arrs]
        cols = [a.shape[2] for a in arrs]
    ranks = [arrs[0].shape[0]] + [a.shape[-1] for a in arrs]
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<II", d, 0 if vector else 1))
        f.write(struct.pack(f"<{d}I", *rows))
        f.write(struct.pack(f"<{d}I", *cols))
        f.write(struct.pack(f"<{d + 1}I", *ranks))
        for a in arrs:
            f.write(a.tobytes(order="C"))


def load(path):
    """Return (kind, ranks, cores): kind "operator" with cores (r, m, n, r') or
    "vector" with cores (r, m, r').  Raises ValueError on any size mismatch."""
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 12 or data[:4] != MAGIC:
        raise ValueError("not a TTB1 file (bad magic)")
    d, flag = struct.unpack_from("<II", data, 4)
    if d < 1 or flag not in (0, 1):
        raise ValueError(f"bad TTB1 header: d={d}, flag={flag}")
    off = 12
    need = off + 4 * (3 * d + 1)
    if len(data) < need:
        raise ValueError("truncated TTB1 header")
    rows = list(struct.unpack_from(f"<{d}I", data, off))
    cols = list(struct.unpack_from(f"<{d}I", data, off + 4 * d))
    ranks = list(struct.unpack_from(f"<{d + 1}I", data, off + 8 * d))
    off = need
    if flag == 0 and any(c != 1 for c in cols):
        raise ValueError("TTB1 vector with column modes != 1")
    if ranks[0] != 1 or ranks[d] != 1 or min(ranks) < 1:
        raise ValueError(f"bad TTB1 ranks {ranks}")
    sizes = [ranks[k] * rows[k] * cols[k] * ranks[k + 1] for k in range(d)]
    if len(data) != off + 8 * sum(sizes):
        raise ValueError(f"TTB1 payload is {len(data) - off} bytes, header implies {8 * sum(sizes)}")
    cores = []
    for k in range(d):
        a = np.frombuffer(data, dtype="<f8", count=sizes[k], offset=off).astype(np.float64)
        off += 8 * sizes[k]
        if flag == 1:
            cores.append(a.reshape(ranks[k], rows[k], cols[k], ranks[k + 1]))
        else:
            cores.append(a.reshape(ranks[k], rows[k], ranks[k + 1]))
    return ("operator" if flag == 1 else "vector"), ranks, cores


def load_operator(path):
    """(ranks, cores) of a binary-mode QTT operator file, ready for QttOperator."""
    kind, ranks, cores = load(path)
    if kind != "operator":
        raise ValueError("TTB1 file holds a vector, not an operator")
    if any(c.shape[1] != 2 or c.shape[2] != 2 for c in cores):
        raise ValueError("only binary modes (m_k = n_k = 2) are supported (DESIGN.md R14)")
    return ranks, cores
