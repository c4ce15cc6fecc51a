"""Seeded synthetic inputs for the QTT apply y = A x (shared by oracle tests,
GPU parity tests and bench.py).

This module draws random numbers and builds core arrays; it holds none of the
apply's arithmetic (no contraction, no sweep).  Both the CPU oracle
(`oracle/`) and the CUDA path (`paper_1511_06029_b200/`) consume what it
returns; neither imports the other.

Conventions (SURVEY.md §8 readings R1, R2, R5-R8):

* A QTT matrix over N = 2**d is a list of d cores ``G[k]`` of shape
  ``(r[k], 2, 2, r[k+1])`` (0-based list index k is the paper's core k+1),
  float64, C order ``[alpha_{k-1}][i_k][j_k][alpha_k]`` with ``i_k`` the
  row/target digit and ``j_k`` the column/source digit (PAPER.md P:953-962,
  "G_k(alpha_{k-1}, overline{i_k j_k}, alpha_k)").
* ``ranks = [r_0, ..., r_d]`` with ``r_0 = r_d = 1``.
* Core 1 acts on bit 0 (the least significant bit) of the row/column index:
  ``i = sum_k i_k 2**(k-1)`` (finest level first).
* x is column-major ``N x nrhs`` (ld = N); as a numpy array it is returned
  with shape ``(nrhs, N)`` in C order, i.e. row s is right-hand side s and the
  memory image is exactly the column-major matrix.
"""
from .configs import CONFIGS, Config, make_config, config_ranks, flops_per_apply
from .gen import generate, random_cores, random_case, rank_profile_random, random_tt_vector, bie_case
from . import closed_forms

__all__ = [
    "CONFIGS", "Config", "make_config", "config_ranks", "flops_per_apply",
    "generate", "random_cores", "random_case", "rank_profile_random", "random_tt_vector", "bie_case",
    "closed_forms",
]
