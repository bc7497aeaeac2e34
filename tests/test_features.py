"""Row features (pkg/src/mpcg/features.py).

CPU: the oracle restatement (oracle/features_oracle.py) against the golden
fixtures produced by running the reference (tests/golden/
make_features_golden.py), bit for bit; the drop-in module's argument checks.
GPU: paper_2407_15973_b200.features (libmpbjac.so) against the same
fixtures bit for bit, and against the oracle on larger matrices.
"""
import os

import numpy as np
import pytest

from oracle import features_oracle as FO

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def fg():
    return np.load(os.path.join(HERE, "golden", "features_golden.npz"))


def _csr(fg, name):
    return fg[f"{name}/row_ptr"], fg[f"{name}/col_idx"], fg[f"{name}/values"]


def _same(a, b):
    """Bitwise equality of float results (NaN == NaN)."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


def _golden_sign(fg, name, tol):
    key = f"{name}/sign_{tol:g}"
    return (tuple(bool(x) for x in fg[key + "/flags"]), fg[key + "/diag"], fg[key + "/offdiag"],
            fg[key + "/rowsum"])


def test_oracle_matches_reference_golden(fg):
    for name in fg["names"]:
        rp, ci, va = _csr(fg, name)
        tau, defined = FO.multiscale_profile(rp, ci, va)
        assert _same(tau, fg[f"{name}/tau"]), name
        assert np.array_equal(defined, fg[f"{name}/defined"]), name
        for key, edges in (("decade", tuple(10.0 ** e for e in range(17))),
                           ("small", (1.0, 2.0, 4.0, 10.0, 100.0, 1000.0))):
            counts, undef = FO.histogram(tau, defined, edges)
            assert counts + (undef,) == tuple(fg[f"{name}/hist_{key}"]), (name, key)
        assert _same(FO.dominance(rp, ci, va), fg[f"{name}/dominance"]), name
        for tol in (0.0, 1e-12):
            flags, d, o, r = FO.sign_check(rp, ci, va, tol)
            gflags, gd, go, gr = _golden_sign(fg, name, tol)
            assert flags == gflags, (name, tol)
            assert _same(np.array(d, np.float64).reshape(-1, 2), gd), (name, tol)
            assert _same(np.array(o, np.float64).reshape(-1, 3), go), (name, tol)
            assert _same(np.array(r, np.float64).reshape(-1, 2), gr), (name, tol)


def test_argument_checks_match_reference():
    from paper_2407_15973_b200 import features as F
    from paper_2407_15973_b200.sparse import SparseMatrix
    A = SparseMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 2.0]))
    for edges, msg in (((), "at least one"), ((1.0, np.inf), "finite"), ((1.0, 1.0), "ascending"),
                       ((2.0, 3.0), "must not exceed 1")):
        with pytest.raises(ValueError, match=msg):
            F.multiscale_histogram(A, edges)
    with pytest.raises(IndexError):
        F.row_multiscale(A, 2)
    assert F.row_multiscale(A, 0) is None
    E = SparseMatrix(0, 0, np.array([0]), np.array([], np.int32), np.array([]))
    for fn in (F.multiscale_profile, F.dominance_stats, F.m_matrix_sign_check):
        with pytest.raises(ValueError, match="no rows"):
            fn(E)
    with pytest.raises(ValueError, match="nonnegative"):
        F.m_matrix_sign_check(A, -1.0)


def _matrix(rp, ci, va):
    from paper_2407_15973_b200.sparse import SparseMatrix
    return SparseMatrix.trusted(rp.size - 1, rp.size - 1, rp, ci, va)


def _check_all(A, rp, ci, va, expect=None):
    """GPU features of A against expect (golden) or the oracle."""
    from paper_2407_15973_b200 import features as F
    tau, defined = F.multiscale_profile(A)
    otau, odef = FO.multiscale_profile(rp, ci, va)
    assert _same(tau, otau) and np.array_equal(defined, odef)
    for edges in (F.DECADE_EDGES, F.SMALL_RATIO_EDGES):
        h = F.multiscale_histogram(A, edges)
        assert (h.counts, h.undefined_count) == FO.histogram(otau, odef, edges)
        assert h.total_rows == A.n
    d = F.dominance_stats(A)
    got = (d.dominance_min, d.dominance_median, d.dominance_max, d.fraction_dominant, d.row_sum_min,
           d.row_sum_max)
    assert _same(got, FO.dominance(rp, ci, va)), (got, FO.dominance(rp, ci, va))
    for tol in (0.0, 1e-12):
        s = F.m_matrix_sign_check(A, tol)
        flags, sd, so, sr = FO.sign_check(rp, ci, va, tol)
        assert (s.diag_positive, s.offdiag_nonpositive, s.row_sums_nonnegative) == flags
        assert s.all_pass == all(flags)
        assert _same(np.array(s.diag_samples, np.float64).reshape(-1, 2), np.array(sd, np.float64).reshape(-1, 2))
        assert _same(np.array(s.offdiag_samples, np.float64).reshape(-1, 3),
                     np.array(so, np.float64).reshape(-1, 3))
        assert _same(np.array(s.row_sum_samples, np.float64).reshape(-1, 2),
                     np.array(sr, np.float64).reshape(-1, 2))
    return tau


@pytest.mark.gpu
def test_features_bitwise_vs_reference_golden(fg, cuda):
    for name in fg["names"]:
        rp, ci, va = _csr(fg, name)
        tau = _check_all(_matrix(rp, ci, va), rp, ci, va)
        assert _same(tau, fg[f"{name}/tau"]), name      # and the reference's own output
        from paper_2407_15973_b200 import features as F
        d = F.dominance_stats(_matrix(rp, ci, va))
        assert _same((d.dominance_min, d.dominance_median, d.dominance_max, d.fraction_dominant,
                      d.row_sum_min, d.row_sum_max), fg[f"{name}/dominance"]), name


@pytest.mark.gpu
def test_features_larger_matrices_vs_oracle(cuda):
    """A config operator (C3 analogue, 32^3: tau spans decades), a random
    matrix with rows of up to 600 entries (all of numpy's summation
    branches) and many sign violations, in fp64 and fp32."""
    from paper_2407_15973_b200 import problems
    cs = problems.make_config("c3", 32)
    A = cs.A
    _check_all(A, A.row_ptr, A.col_idx, A.values)
    rng = np.random.default_rng(11)
    n = 3000
    lens = rng.choice([0, 1, 2, 7, 8, 9, 64, 127, 128, 129, 130, 255, 256, 257, 600], size=n)
    rows, cols = [], []
    for i, m in enumerate(lens):
        cs_ = np.sort(rng.choice(n, size=int(m), replace=False))
        rows.append(np.full(cs_.size, i))
        cols.append(cs_)
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    vals = rng.standard_normal(rows.size) * 10.0 ** rng.integers(-8, 8, rows.size)
    vals[rng.random(rows.size) < 0.05] = 0.0
    rp = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    for dt in (np.float64, np.float32):
        va = vals.astype(dt)
        _check_all(_matrix(rp, cols.astype(np.int32), va), rp, cols.astype(np.int32), va)
