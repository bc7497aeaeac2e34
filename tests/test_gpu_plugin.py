"""The reference's kernel plugin seam, served by libmpbjac.so.

``paper_2407_15973_b200.kernels_b200`` has the signatures of the reference's
``mpcg.kernels_numba`` (pkg/src/mpcg/kernels_numba.py:15-115) and
``backend.use_backend`` mirrors pkg/src/mpcg/backend.py:17-30, the seam the
reference's ``any_backend`` fixture monkeypatches (pkg/tests/conftest.py:8-17).
Every function is checked here against the reference's golden fixtures and
the CPU oracle (which restates kernels_numba.py and is pinned to it), bit for
bit, including explicit in_block masks that are not block-shaped and partial
row ranges, as block_jacobi_sweeps allows.
"""
import numpy as np
import pytest

from conftest import golden_cases, random_spd_csr

pytestmark = pytest.mark.gpu


def _mat(g, name):
    return g[f"{name}/row_ptr"], g[f"{name}/col_idx"], g[f"{name}/values"]


def test_use_backend_binds_b200(cuda):
    from paper_2407_15973_b200 import backend, kernels_b200
    assert backend.use_backend("b200") is kernels_b200
    assert backend.kernels is kernels_b200 and backend.name == "b200"
    for other in ("numba", "numpy", "cpu"):
        with pytest.raises(ValueError, match="unknown backend"):
            backend.use_backend(other)
    assert backend.kernels is kernels_b200
    assert kernels_b200.reduction_mode == "tree"


def test_csr_matvec_plugin_bitwise(golden, cuda):
    from paper_2407_15973_b200 import backend
    K = backend.use_backend("b200")
    for name in golden_cases(golden):
        rp, ci, v = _mat(golden, name)
        n = rp.size - 1
        x = np.cos(np.arange(n) * 0.37)
        out = np.full(n, np.nan)
        K.csr_matvec(rp, ci, v, x, out)
        np.testing.assert_array_equal(out, golden[f"{name}/spmv64"], err_msg=name)
        out32 = np.full(n, np.nan, np.float32)
        K.csr_matvec(rp, ci, v.astype(np.float32), x.astype(np.float32), out32)
        np.testing.assert_array_equal(out32, golden[f"{name}/spmv32"], err_msg=name)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("t", [1, 2, 3])
def test_block_jacobi_sweeps_plugin_masks_and_ranges(golden, cuda, oracle, dtype, t):
    """Arbitrary in_block masks (block-derived, random, all-true, none) and
    partial row ranges, y / tmp updated in place exactly like the oracle's
    restatement of kernels_numba.py:48-70."""
    from paper_2407_15973_b200 import backend
    K = backend.use_backend("b200")
    rng = np.random.default_rng(11 + t)
    for name in ("rspd200", "c2_n16", "c4_n6", "dis10"):
        rp, ci, v = _mat(golden, name)
        n = rp.size - 1
        vals = v.astype(dtype)
        rows = np.repeat(np.arange(n), np.diff(rp))
        diag = np.zeros(n, dtype)
        hit = ci == rows
        diag[rows[hit]] = vals[hit]
        offs = golden[f"{name}/pcg/offsets"]
        blk = np.searchsorted(offs, np.arange(n), side="right") - 1
        masks = {
            "blocks": blk[rows] == blk[ci],
            "random": rng.uniform(size=ci.size) < 0.6,
            "all": np.ones(ci.size, bool),
            "none": np.zeros(ci.size, bool),
        }
        r = (golden[f"{name}/r"]).astype(dtype)
        for mname, mask in masks.items():
            for lo, hi in ((0, n), (n // 3, n - n // 5), (7, 8), (5, 5)):
                y0 = rng.standard_normal(n).astype(dtype)      # rows outside [lo, hi) keep these
                tmp0 = rng.standard_normal(n).astype(dtype)
                yg, tg = y0.copy(), tmp0.copy()
                yo, to = y0.copy(), tmp0.copy()
                K.block_jacobi_sweeps(rp, ci, vals, mask, diag, t, r, yg, tg, lo, hi)
                oracle.block_jacobi_sweeps(rp, ci, vals, mask, diag, t, r, yo, to, lo, hi)
                np.testing.assert_array_equal(yg, yo, err_msg=f"{name} {mname} [{lo},{hi})")
                np.testing.assert_array_equal(tg, to, err_msg=f"{name} {mname} [{lo},{hi}) tmp")


def test_block_jacobi_sweeps_plugin_hand_values(cuda):
    """Hand-derived sweeps.  The reference's A = [[2,-1],[-1,2]], one block,
    r = (1,1) (pkg/tests/test_bjac.py:116-121): y = 1/2, 3/4, 7/8 after
    t = 1, 2, 3.  And an off-diagonal-only mask on [[4,1],[1,4]]: y = 1/4,
    then y += (1 - y)/4: 7/16, 37/64."""
    from paper_2407_15973_b200 import kernels_b200 as K
    rp = np.array([0, 2, 4])
    ci = np.array([0, 1, 0, 1], np.int32)
    cases = ((np.array([2.0, -1.0, -1.0, 2.0]), np.ones(4, bool), (0.5, 0.75, 0.875)),
             (np.array([4.0, 1.0, 1.0, 4.0]), np.array([False, True, True, False]),
              (0.25, 0.4375, 0.578125)))
    for v, mask, wants in cases:
        diag = v[[0, 3]].copy()
        for dt in (np.float64, np.float32):
            for t, want in zip((1, 2, 3), wants):
                y, tmp = np.zeros(2, dt), np.zeros(2, dt)
                K.block_jacobi_sweeps(rp, ci, v.astype(dt), mask, diag.astype(dt), t,
                                      np.ones(2, dt), y, tmp, 0, 2)
                np.testing.assert_array_equal(y, [want, want])


def test_dot_and_norm_plugin(cuda, oracle):
    from paper_2407_15973_b200 import kernels_b200 as K
    rng = np.random.default_rng(3)
    for n in (0, 1, 255, 256, 257, 100_003):
        a, b = rng.standard_normal(n), rng.standard_normal(n)
        tiles = np.append(np.arange(0, n, 256), n) if n else np.array([0])
        got = K.dot_seq(a, b)
        assert isinstance(got, np.float64)
        if n:
            assert got == oracle.tree_dot(tiles, a, b)           # device order, bitwise
            assert got == pytest.approx(oracle.dot_seq(a, b), rel=1e-12, abs=1e-12)
        else:
            assert got == 0.0
        g32 = K.dot_seq(a.astype(np.float32), b.astype(np.float32))
        assert isinstance(g32, np.float32)
        if n:
            assert g32 == pytest.approx(float(np.dot(a, b)), rel=1e-4, abs=1e-3)
        nrm = K.norm_sq_f64(a)
        assert nrm == pytest.approx(oracle.norm_sq_f64(a), rel=1e-13, abs=0)
        nrm32 = K.norm_sq_f64(a.astype(np.float32))
        assert nrm32 == pytest.approx(oracle.norm_sq_f64(a.astype(np.float32)), rel=1e-13, abs=0)


def test_fill_stencil_plugin(golden, cuda):
    """fill_stencil (kernels_numba.py:73-115) reproduces the reference's
    assembly of the const8 fixture (built by the reference's build_matrix)."""
    from paper_2407_15973_b200 import kernels_b200 as K, problems
    rp, ci, v = _mat(golden, "const8")
    n = 8
    faces = problems.face_arrays(np.ones(n ** 3).reshape(n, n, n))
    col = np.empty_like(ci)
    val = np.empty_like(v)
    K.fill_stencil(n, *faces, float((n + 1) ** 2), rp, col, val)
    np.testing.assert_array_equal(col, ci)
    np.testing.assert_array_equal(val, v)


def test_plugin_random_spd_matvec(cuda, oracle):
    """A random SPD CSR (pkg/tests/conftest.py:28-34 recipe) through the
    plugin matvec, fp64 and fp32, vs the oracle."""
    from paper_2407_15973_b200 import kernels_b200 as K
    rng = np.random.default_rng(9)
    A = random_spd_csr(300, 0.1, rng)
    x = rng.standard_normal(300)
    for dt in (np.float64, np.float32):
        got, want = np.empty(300, dt), np.empty(300, dt)
        K.csr_matvec(A.row_ptr, A.col_idx, A.values.astype(dt), x.astype(dt), got)
        oracle.csr_matvec(A.row_ptr, A.col_idx, A.values.astype(dt), x.astype(dt), want)
        np.testing.assert_array_equal(got, want)
