"""Generate tests/golden/features_golden.npz by running the REFERENCE's
features module (pkg/src/mpcg/features.py) on fixed matrices.

Run in the build container (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_features_golden.py

Matrices: every matrix of golden.npz (the reference's own const/ani/dis/rand
families and the config analogues), plus hand-made edge cases (empty,
diagonal-only and explicit-zero rows, one qualifying entry, NaN / inf
entries, positive off-diagonals, missing diagonals, negative row sums, fp32
values) and a random matrix with rows of up to 300 entries (numpy's
pairwise-summation branches).  Recorded per matrix: multiscale_profile,
multiscale_histogram for both edge sets, dominance_stats, and
m_matrix_sign_check at two tolerances.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from mpcg import features as F  # noqa: E402  (the reference)
from mpcg.sparse import SparseMatrix as RefMatrix  # noqa: E402


def edge_cases():
    """(name, n, rows, cols, vals, dtype) COO edge cases."""
    out = []
    # 0 empty row, 1 diagonal only, 2 explicit-zero off-diagonals, 3 one qualifying
    # entry, 4 NaN entry, 5 inf entry, 6 positive off-diagonal, 7 no diagonal,
    # 8 negative row sum, 9 zero diagonal
    r = [1, 2, 2, 2, 3, 3, 3, 4, 4, 4, 5, 5, 6, 6, 6, 7, 7, 8, 8, 8, 9, 9]
    c = [1, 1, 2, 3, 2, 3, 4, 3, 4, 5, 4, 5, 5, 6, 7, 6, 8, 7, 8, 9, 8, 9]
    v = [2.0, 0.0, 3.0, 0.0, -1.0, 4.0, -1e-3, np.nan, 5.0, -2.0, np.inf, 1.0, 0.5, 3.0, -1.0,
         -2.0, -1.0, -3.0, 1.0, -0.5, -1.0, 0.0]
    out.append(("edges64", 10, r, c, v, np.float64))
    out.append(("edges32", 10, r, c, v, np.float32))
    # an M-matrix that passes, and one with many violations (more than 10 of each)
    n = 40
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i); cols.append(i); vals.append(4.0)
        for j in (i - 1, i + 1):
            if 0 <= j < n:
                rows.append(i); cols.append(j); vals.append(-1.0)
    out.append(("mmat_ok", n, rows, cols, vals, np.float64))
    vals_bad = [(-v if (k % 3 == 0) else v * 3.0) for k, v in enumerate(vals)]
    out.append(("mmat_bad", n, rows, cols, vals_bad, np.float64))
    return out


def long_rows(seed=7, n=160):
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        m = int(rng.choice([1, 3, 7, 8, 9, 15, 16, 17, 100, 128, 129, 130, 200, 257, 300]))
        m = min(m, n)
        cs = np.sort(rng.choice(n, size=m, replace=False))
        if i not in cs:
            cs[rng.integers(m)] = i
            cs = np.sort(cs)
        for c in cs:
            rows.append(i); cols.append(int(c))
            vals.append(float(rng.standard_normal() * 10.0 ** rng.integers(-6, 6)))
    return rows, cols, vals


def record(out, name, A):
    tau, defined = F.multiscale_profile(A)
    out[f"{name}/tau"] = tau
    out[f"{name}/defined"] = defined
    for key, edges in (("decade", F.DECADE_EDGES), ("small", F.SMALL_RATIO_EDGES)):
        hst = F.multiscale_histogram(A, edges)
        out[f"{name}/hist_{key}"] = np.array(hst.counts + (hst.undefined_count,), np.int64)
    d = F.dominance_stats(A)
    out[f"{name}/dominance"] = np.array([d.dominance_min, d.dominance_median, d.dominance_max,
                                         d.fraction_dominant, d.row_sum_min, d.row_sum_max])
    for tol in (0.0, 1e-12):
        s = F.m_matrix_sign_check(A, tol)
        key = f"{name}/sign_{tol:g}"
        out[key + "/flags"] = np.array([s.diag_positive, s.offdiag_nonpositive, s.row_sums_nonnegative])
        out[key + "/diag"] = np.array(s.diag_samples, np.float64).reshape(-1, 2)
        out[key + "/offdiag"] = np.array(s.offdiag_samples, np.float64).reshape(-1, 3)
        out[key + "/rowsum"] = np.array(s.row_sum_samples, np.float64).reshape(-1, 2)


def main():
    g = np.load(os.path.join(HERE, "golden.npz"))
    out = {}
    names = []
    for key in g.files:
        if key.endswith("/row_ptr"):
            name = key[:-len("/row_ptr")]
            rp, ci, va = g[f"{name}/row_ptr"], g[f"{name}/col_idx"], g[f"{name}/values"]
            n = rp.size - 1
            A = RefMatrix(n, n, rp.astype(np.int64), ci.astype(np.int32), va.astype(np.float64))
            out[f"{name}/row_ptr"], out[f"{name}/col_idx"], out[f"{name}/values"] = A.row_ptr, A.col_idx, A.values
            record(out, name, A)
            names.append(name)
    cases = edge_cases() + [("long_rows", 160) + tuple(long_rows()) + (np.float64,)]
    for name, n, r, c, v, dt in cases:
        A = RefMatrix.from_coo(n, n, np.asarray(r), np.asarray(c), np.asarray(v, np.float64), dtype=dt)
        out[f"{name}/row_ptr"], out[f"{name}/col_idx"], out[f"{name}/values"] = A.row_ptr, A.col_idx, A.values
        record(out, name, A)
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "features_golden.npz"), **out)
    print(f"wrote {len(names)} matrices to features_golden.npz")


if __name__ == "__main__":
    main()
