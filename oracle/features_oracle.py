"""CPU restatement of the reference's row features (test infrastructure).

TEST INFRASTRUCTURE ONLY: imported by tests/ as the checker of the GPU
features (paper_2407_15973_b200/features.py); never by the product path.

Restates pkg/src/mpcg/features.py:27-211 with numpy on host arrays
(row_ptr int64, col_idx, values): the per-row sums use np.add.reduceat
exactly as the reference does (features.py:31-38), so results are the
reference's bit for bit; pinned to fixtures produced by running the
reference (tests/golden/make_features_golden.py).
"""
from __future__ import annotations

import numpy as np


def _rows(row_ptr):
    return np.repeat(np.arange(row_ptr.size - 1), np.diff(row_ptr))


def _reduce_rows(values, row_ptr, fill, ufunc):          # features.py:31-38
    n = row_ptr.size - 1
    out = np.full(n, fill)
    nonempty = np.flatnonzero(row_ptr[:-1] != row_ptr[1:])
    if nonempty.size:
        out[nonempty] = ufunc.reduceat(values, row_ptr[nonempty])
    return out


def _diagonal(row_ptr, col_idx, values):                  # sparse.py diagonal()
    rows = _rows(row_ptr)
    d = np.zeros(row_ptr.size - 1, dtype=values.dtype)
    on = rows == col_idx
    d[rows[on]] = values[on]
    return d


def multiscale_profile(row_ptr, col_idx, values):         # features.py:41-55
    rows = _rows(row_ptr)
    absv = np.abs(values).astype(np.float64)
    qual = (rows != col_idx) & (values != 0)
    row_max = _reduce_rows(np.where(qual, absv, -np.inf), row_ptr, -np.inf, np.maximum)
    row_min = _reduce_rows(np.where(qual, absv, np.inf), row_ptr, np.inf, np.minimum)
    defined = np.isfinite(row_max)
    tau = np.full(row_ptr.size - 1, np.nan)
    tau[defined] = row_max[defined] / row_min[defined]
    return tau, defined


def histogram(tau, defined, edges):                       # features.py:94-113
    arr = np.asarray(edges, np.float64)
    idx = np.searchsorted(arr, tau[defined], side="right") - 1
    counts = np.bincount(idx, minlength=len(edges))
    return tuple(int(c) for c in counts), int((~defined).sum())


def dominance(row_ptr, col_idx, values):                  # features.py:127-152
    rows = _rows(row_ptr)
    absv = np.abs(values).astype(np.float64)
    off_sums = _reduce_rows(np.where(rows != col_idx, absv, 0.0), row_ptr, 0.0, np.add)
    diag = np.abs(_diagonal(row_ptr, col_idx, values).astype(np.float64))
    with np.errstate(divide="ignore", invalid="ignore"):
        dom = np.where(off_sums == 0.0, np.inf, diag / off_sums)
    row_sums = _reduce_rows(values.astype(np.float64), row_ptr, 0.0, np.add)
    return (float(dom.min()), float(np.median(dom)), float(dom.max()),
            float(np.mean(dom > 1.0)), float(row_sums.min()), float(row_sums.max()))


def sign_check(row_ptr, col_idx, values, tol=0.0):        # features.py:171-211
    rows = _rows(row_ptr)
    diag = _diagonal(row_ptr, col_idx, values).astype(np.float64)
    bad_diag = np.flatnonzero(~(diag > 0))
    bad_off = np.flatnonzero((rows != col_idx) & (values > 0))
    vals64 = values.astype(np.float64)
    row_sums = _reduce_rows(vals64, row_ptr, 0.0, np.add)
    abs_sums = _reduce_rows(np.abs(vals64), row_ptr, 0.0, np.add)
    with np.errstate(invalid="ignore"):
        bad_sum = np.flatnonzero(row_sums < -(tol * abs_sums))
    return ((bad_diag.size == 0, bad_off.size == 0, bad_sum.size == 0),
            tuple((int(i), float(diag[i])) for i in bad_diag[:10]),
            tuple((int(rows[p]), int(col_idx[p]), float(values[p])) for p in bad_off[:10]),
            tuple((int(i), float(row_sums[i])) for i in bad_sum[:10]))
