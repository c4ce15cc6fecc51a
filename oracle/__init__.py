"""CPU oracle for the QTT apply y = A x  --  TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously correct NumPy (float64 unless a caller passes another
dtype) implementations of what PAPER.md's Alg. 2 computes.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1511_06029_b200``) never imports it and shares no code
with it; the only common module is the seeded input generator
``qtt_workload`` (which holds none of the method's arithmetic).

Every function is pinned by ``tests/test_oracle_pins.py`` against something
other than itself (closed forms, library routines, brute force, invariants);
see DESIGN.md §"Oracle and pins".  No function here is "parity unpinned".
"""
from .qtt_oracle import (
    entry, dense_matrix, apply_dense, apply_bitwise, alg2_sweep, apply_alg2,
    blas_sweep, apply_blas_sweep, top_projection, apply_chunked, kron_apply_modes,
    apply_rows, compose, transpose, compressed_matvec, tt_vector_dense,
    tt_vector_entries, kron_vector_cores,
)
from .checks import compare, assert_close
from . import morton

__all__ = [
    "entry", "dense_matrix", "apply_dense", "apply_bitwise", "alg2_sweep",
    "apply_alg2", "blas_sweep", "apply_blas_sweep", "top_projection", "apply_chunked",
    "kron_apply_modes", "apply_rows", "compose", "transpose", "compressed_matvec",
    "tt_vector_dense", "tt_vector_entries", "kron_vector_cores", "compare", "assert_close", "morton",
]
