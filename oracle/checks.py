"""Error metrics for GPU-vs-oracle parity  --  TEST INFRASTRUCTURE ONLY.

Tolerances (BASELINE.json north_star; reading R11 in DESIGN.md):
  * relative l2 per RHS column:  ||yhat - y||_2 / ||y||_2 <= 1e-12
  * elementwise relative error with an RMS floor:
        max_i |yhat_i - y_i| / max(|y_i|, ||y||_2 / sqrt(n)) <= 1e-10
    (two correct fp64 summation orders differ by up to ~1e-8 raw relative
    error on entries where y_i ~ 0 through cancellation; the floor at the RMS
    of the reference column removes exactly those).  The raw elementwise
    relative error and the count of entries above 1e-10 are reported too, and
    every such raw offender must satisfy |y_i| < 1e-3 * RMS.
"""
from __future__ import annotations

import numpy as np

L2_TOL = 1e-12
ELEM_TOL = 1e-10


def compare(yhat, y, rms=None):
    """Per-column metrics. yhat, y: (nrhs, n). ``rms`` overrides the floor
    (used for sampled rows, where it is the RMS of the sampled reference)."""
    yhat = np.atleast_2d(np.asarray(yhat, dtype=np.float64))
    y = np.atleast_2d(np.asarray(y, dtype=np.float64))
    assert yhat.shape == y.shape, (yhat.shape, y.shape)
    res = []
    for s in range(y.shape[0]):
        a, b = yhat[s], y[s]
        n = b.size
        nrm = np.linalg.norm(b)
        fl = (nrm / np.sqrt(n)) if rms is None else rms
        diff = np.abs(a - b)
        rel_l2 = float(np.linalg.norm(a - b) / nrm) if nrm > 0 else float(np.linalg.norm(a - b))
        den = np.maximum(np.abs(b), fl)
        elem_floor = float(np.max(diff / den)) if n else 0.0
        with np.errstate(divide="ignore", invalid="ignore"):
            raw = np.where(b != 0, diff / np.abs(b), np.where(diff == 0, 0.0, np.inf))
        off = np.nonzero(raw > ELEM_TOL)[0]
        res.append(dict(
            rel_l2=rel_l2, elem_floor=elem_floor,
            raw_elem_max=float(np.max(raw)) if n else 0.0,
            raw_offenders=int(off.size),
            offender_max_rel_mag=float(np.max(np.abs(b[off]) / fl)) if off.size else 0.0,
            nan_mismatch=bool(np.any(np.isnan(a) != np.isnan(b))),
        ))
    return res


def assert_close(yhat, y, rms=None, l2_tol=L2_TOL, elem_tol=ELEM_TOL, check_l2=True):
    for s, m in enumerate(compare(yhat, y, rms)):
        assert not m["nan_mismatch"], (s, m)
        if check_l2:
            assert m["rel_l2"] <= l2_tol, (s, m)
        assert m["elem_floor"] <= elem_tol, (s, m)
        assert m["offender_max_rel_mag"] < 1e-3, (s, m)
    return True
