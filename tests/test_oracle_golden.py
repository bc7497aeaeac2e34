"""Pin the CPU oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py).  Everything here is bit-exact: the oracle in
sequential mode IS the reference's arithmetic, including its dot order."""
import numpy as np
import pytest

from conftest import golden_cases

KT = ((1, 1), (1, 2), (2, 2), (2, 3), (3, 2))
POLICIES = ("uniform", "fixed-low", "adaptive-hl:10", "adaptive-lh:1e-5", "adaptive-hl:1e-3")


def _parts(g, name):
    return sorted({k.split("/")[1] for k in g if k.startswith(name + "/")
                   and k.endswith("/offsets")} - {"pcg"})


def _mat(g, name):
    return g[f"{name}/row_ptr"], g[f"{name}/col_idx"], g[f"{name}/values"]


def test_golden_covers_expected_cases(golden):
    names = golden_cases(golden)
    for want in ("rspd40", "rspd200", "const8", "ani6", "dis10", "rand12",
                 "c1_n16", "c2_n16", "c3_n16", "c4_n6", "c5_n16"):
        assert want in names


def test_spmv_bitwise(golden, oracle):
    for name in golden_cases(golden):
        rp, ci, v = _mat(golden, name)
        n = rp.size - 1
        x = np.cos(np.arange(n) * 0.37)
        out = np.empty(n)
        oracle.csr_matvec(rp, ci, v, x, out)
        np.testing.assert_array_equal(out, golden[f"{name}/spmv64"])
        out32 = np.empty(n, np.float32)
        oracle.csr_matvec(rp, ci, v.astype(np.float32), x.astype(np.float32), out32)
        np.testing.assert_array_equal(out32, golden[f"{name}/spmv32"])


def test_bjac_apply_bitwise(golden, oracle):
    checked = 0
    for name in golden_cases(golden):
        rp, ci, v = _mat(golden, name)
        r = golden[f"{name}/r"]
        for pname in _parts(golden, name):
            offs = golden[f"{name}/{pname}/offsets"]
            d64, d32, v32, inb = oracle.setup_arrays(rp, ci, v, offs)
            for k, t in KT:
                z64 = oracle.bjac_apply(rp, ci, v, inb, d64, k, t, r)
                np.testing.assert_array_equal(z64, golden[f"{name}/{pname}/apply_f64_k{k}t{t}"])
                z32 = oracle.bjac_apply(rp, ci, v32, inb, d32, k, t, r.astype(np.float32))
                np.testing.assert_array_equal(z32, golden[f"{name}/{pname}/apply_f32_k{k}t{t}"])
                checked += 2
    assert checked > 100


def test_fmp_apply_bitwise(golden, oracle):
    for name in golden_cases(golden):
        rp, ci, v = _mat(golden, name)
        r = golden[f"{name}/r"]
        for pname in _parts(golden, name):
            offs = golden[f"{name}/{pname}/offsets"]
            _, d32, v32, inb = oracle.setup_arrays(rp, ci, v, offs)
            r32, cnt, _ = oracle.narrow(r)
            assert cnt == 0
            z = oracle.bjac_apply(rp, ci, v32, inb, d32, 2, 2, r32).astype(np.float64)
            np.testing.assert_array_equal(z, golden[f"{name}/{pname}/fmp_k2t2"])


@pytest.mark.parametrize("pol", POLICIES)
def test_pcg_sequential_matches_reference_bitwise(golden, oracle, pol):
    for name in golden_cases(golden):
        rp, ci, v = _mat(golden, name)
        offs = golden[f"{name}/pcg/offsets"]
        key = f"{name}/pcg/{pol}"
        tol, k, t = golden[f"{key}/meta"]
        kind, _, tolstr = pol.partition(":")
        out = oracle.pcg_solve(rp, ci, v, golden[f"{name}/b"], offs, kind=kind,
                               adp_tol=float(tolstr) if tolstr else None, k=int(k), t=int(t),
                               res_tol=tol, stride=5, order="sequential")
        assert out["iterations"] == int(golden[f"{key}/iterations"]), name
        assert out["converged"] == bool(golden[f"{key}/converged"])
        np.testing.assert_array_equal(out["relres"], golden[f"{key}/relres"])
        np.testing.assert_array_equal(np.array(out["branch"]) == "low",
                                      golden[f"{key}/branch"].astype(bool))
        np.testing.assert_array_equal(out["x"], golden[f"{key}/x"])
        assert out["final_true_relres"] == float(golden[f"{key}/final_true"])
        # strided true residuals (the last entry is filled in by pcg_solve
        # itself when it converged, solver.py:179-182)
        np.testing.assert_array_equal(out["true_relres"], golden[f"{key}/true"])


def test_device_order_differs_only_in_dots(golden, oracle):
    """The device-order replay changes only the dot summation order: same
    iteration counts on every golden case (these are not delay regimes)."""
    for name in ("c1_n16", "c2_n16", "c3_n16", "c5_n16", "const8", "rand12"):
        rp, ci, v = _mat(golden, name)
        offs = golden[f"{name}/pcg/offsets"]
        tol, k, t = golden[f"{name}/pcg/fixed-low/meta"]
        out = oracle.pcg_solve(rp, ci, v, golden[f"{name}/b"], offs, kind="fixed-low",
                               k=int(k), t=int(t), res_tol=tol, order="device")
        assert abs(out["iterations"] - int(golden[f"{name}/pcg/fixed-low/iterations"])) <= 2


AUG_POLICIES = ("fixed-low", "uniform", "adaptive-hl:1e-3", "adaptive-lh:1e-4")


@pytest.fixture(scope="module")
def augment_golden():
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "augment_golden.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("pol", AUG_POLICIES)
def test_oracle_preconditioner_from_other_matrix(augment_golden, oracle, pol):
    """pcg_solve(A, b, build_mixed(diag_augment(A, p), ..)): the reference
    multiplies by A and preconditions with the augmented values
    (tests/golden/make_augment_golden.py); the oracle's prec_values path
    reproduces it bit for bit."""
    g = augment_golden
    from paper_2407_15973_b200 import SparseMatrix
    from paper_2407_15973_b200.problems import diag_augment
    for name in sorted({k.split("/")[0] for k in g}):
        rp, ci, v, pv = (g[f"{name}/{s}"] for s in ("row_ptr", "col_idx", "values", "prec_values"))
        pd, k, t, tol = g[f"{name}/meta"]
        mine = diag_augment(SparseMatrix(rp.size - 1, rp.size - 1, rp, ci, v), float(pd))
        np.testing.assert_array_equal(mine.values, pv)
        kind, _, tolstr = pol.partition(":")
        out = oracle.pcg_solve(rp, ci, v, g[f"{name}/b"], g[f"{name}/offsets"], kind=kind,
                               adp_tol=float(tolstr) if tolstr else None, k=int(k), t=int(t),
                               res_tol=tol, stride=4, order="sequential", prec_values=pv)
        key = f"{name}/{pol}"
        assert out["iterations"] == int(g[f"{key}/iterations"]), name
        np.testing.assert_array_equal(out["relres"], g[f"{key}/relres"])
        np.testing.assert_array_equal(out["x"], g[f"{key}/x"])
        np.testing.assert_array_equal(out["true_relres"], g[f"{key}/true"])
        assert out["final_true_relres"] == float(g[f"{key}/final_true"])
