"""GPU parity: libmpbjac.so against the reference's golden fixtures and the
CPU oracle, through the drop-in API (which calls the C-ABI).

Bit-exact expectations (thread-per-row, no FMA, IEEE division):
  spmv, BjacPreconditioner.apply (fp64 and fp32, every partition regime,
  every (k, t)), fmp_apply, inner_apply, narrowing;  whole PCG solves vs the
  oracle's device-order replay (x, trace, branches, iteration count).
Band expectations: PCG iteration counts vs the reference's own sequential
dot order within max(2, envelope).
"""
import numpy as np
import pytest

from conftest import dense_to_csr, golden_cases, random_spd_csr

pytestmark = pytest.mark.gpu

KT = ((1, 1), (1, 2), (2, 2), (2, 3), (3, 2))
POLICIES = ("uniform", "fixed-low", "adaptive-hl:10", "adaptive-lh:1e-5", "adaptive-hl:1e-3")


def _parts(g, name):
    return sorted({k.split("/")[1] for k in g if k.startswith(name + "/")
                   and k.endswith("/offsets")} - {"pcg"})


def _matrix(g, name):
    from paper_2407_15973_b200 import SparseMatrix
    rp = g[f"{name}/row_ptr"]
    return SparseMatrix(rp.size - 1, rp.size - 1, rp, g[f"{name}/col_idx"], g[f"{name}/values"])


def test_spmv_bitwise(golden, cuda):
    from paper_2407_15973_b200 import Precision, convert_precision, spmv
    for name in golden_cases(golden):
        A = _matrix(golden, name)
        x = np.cos(np.arange(A.n) * 0.37)
        np.testing.assert_array_equal(spmv(A, x), golden[f"{name}/spmv64"])
        A32 = convert_precision(A, Precision.F32)
        np.testing.assert_array_equal(spmv(A32, x.astype(np.float32)), golden[f"{name}/spmv32"])


def test_bjac_apply_bitwise_all_regimes(golden, cuda):
    """Small blocks (fused smem kernel), nb=32 / nb=2 / nb=1 large blocks
    (multi-launch path), 96-row 3-T blocks; fp64 and fp32; k,t up to 3."""
    from paper_2407_15973_b200 import Precision
    from paper_2407_15973_b200.bjac import BlockPartition, setup
    n_checked = 0
    for name in golden_cases(golden):
        A = _matrix(golden, name)
        r = golden[f"{name}/r"]
        for pname in _parts(golden, name):
            part = BlockPartition(golden[f"{name}/{pname}/offsets"])
            for k, t in KT:
                for prec in (Precision.F64, Precision.F32):
                    P = setup(A, k=k, t=t, precision=prec, partition=part)
                    z = P.apply(r.astype(prec.dtype))
                    assert z.dtype == prec.dtype
                    np.testing.assert_array_equal(
                        z, golden[f"{name}/{pname}/apply_{prec}_k{k}t{t}"],
                        err_msg=f"{name}/{pname} {prec} k={k} t={t}")
                    n_checked += 1
    assert n_checked > 100


def test_fmp_apply_bitwise(golden, cuda):
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed, fmp_apply
    for name in golden_cases(golden):
        A = _matrix(golden, name)
        r = golden[f"{name}/r"]
        for pname in _parts(golden, name):
            part = BlockPartition(golden[f"{name}/{pname}/offsets"])
            mp = build_mixed(A, PrecisionPolicy.parse("fixed-low"), k=2, t=2, partition=part)
            z, br = fmp_apply(mp, r)
            assert br == "low" and z.dtype == np.float64
            np.testing.assert_array_equal(z, golden[f"{name}/{pname}/fmp_k2t2"])


def test_inner_apply_matches_apply_rows(cuda):
    from paper_2407_15973_b200.bjac import setup
    rng = np.random.default_rng(21)
    A = random_spd_csr(30, 0.3, rng)
    P = setup(A, nb=4, k=1, t=3)
    r = rng.standard_normal(30)
    z = P.apply(r)
    for b in range(P.partition.num_blocks):
        s, e = P.partition.block_range(b)
        np.testing.assert_array_equal(P.inner_apply(b, r[s:e]), z[s:e])


def test_hand_derived_known_answers(cuda):
    """pkg/tests/test_bjac.py:116-128 and :155-163."""
    from paper_2407_15973_b200.bjac import setup
    A = dense_to_csr([[2.0, -1.0], [-1.0, 2.0]])
    np.testing.assert_array_equal(setup(A, nb=1, k=1, t=2).apply(np.ones(2)), [0.75, 0.75])
    np.testing.assert_array_equal(setup(A, nb=1, k=2, t=2).apply(np.ones(2)), [0.9375, 0.9375])
    d = np.array([2.0, 0.5, 8.0, 0.25])
    D = dense_to_csr(np.diag(d))
    r = np.array([1.3, -0.7, 2.9, 0.11])
    for k, t in ((1, 3), (2, 2), (3, 1)):
        np.testing.assert_array_equal(setup(D, nb=2, k=k, t=t).apply(r), r / d)


def test_point_jacobi_is_exact_division(cuda):
    """k = t = 1 returns r / diag bit for bit (test_acceptance.py:110-129)."""
    from paper_2407_15973_b200 import Precision
    from paper_2407_15973_b200.bjac import setup
    for seed in range(6):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(5, 40))
        A = random_spd_csr(n, 0.3, rng)
        for prec in (Precision.F64, Precision.F32):
            P = setup(A, nb=min(4, n), k=1, t=1, precision=prec)
            r = rng.standard_normal(n).astype(prec.dtype)
            np.testing.assert_array_equal(P.apply(r), r / A.diagonal().astype(prec.dtype))


def test_linearity_power_of_two(cuda):
    from paper_2407_15973_b200.bjac import setup
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed, fmp_apply
    rng = np.random.default_rng(3)
    A = random_spd_csr(25, 0.3, rng)
    P = setup(A, nb=5, k=2, t=2)
    r = rng.standard_normal(25)
    np.testing.assert_array_equal(P.apply(4.0 * r), 4.0 * P.apply(r))
    mp = build_mixed(A, PrecisionPolicy.parse("fixed-low"), nb=5)
    np.testing.assert_array_equal(fmp_apply(mp, 8.0 * r)[0], 8.0 * fmp_apply(mp, r)[0])


def test_setup_errors_match_reference(cuda):
    from paper_2407_15973_b200 import NarrowingOverflowError, Precision, SparseMatrix
    from paper_2407_15973_b200.bjac import BlockPartition, setup
    with pytest.raises(ValueError, match="square"):
        setup(SparseMatrix.from_coo(2, 3, [0, 1], [0, 1], [1.0, 1.0]), nb=1)
    with pytest.raises(ValueError, match="row 1"):
        setup(SparseMatrix.from_coo(2, 2, [0, 1], [0, 0], [1.0, 1.0]), nb=1)
    with pytest.raises(ValueError, match="zero diagonal entry at row 1"):
        setup(SparseMatrix(2, 2, [0, 1, 2], [0, 1], np.array([1.0, 0.0])), nb=1)
    with pytest.raises(ValueError, match="underflows"):
        setup(dense_to_csr([[1e-50, 0.0], [0.0, 1.0]]), nb=1, precision=Precision.F32)
    with pytest.raises(ValueError, match="split"):
        setup(dense_to_csr(np.eye(3)), nb=4)
    with pytest.raises(ValueError, match="sweep"):
        setup(dense_to_csr(np.eye(3)), nb=1, k=0)
    with pytest.raises(ValueError, match="partition"):
        setup(dense_to_csr(np.eye(3)), partition=BlockPartition([0, 2]))
    with pytest.raises(NarrowingOverflowError):
        setup(dense_to_csr([[1.0, 1e40], [1e40, 1.0]]), nb=1, precision=Precision.F32)


def test_narrowing_and_norms(cuda, oracle):
    from paper_2407_15973_b200 import NarrowingOverflowError, Precision, convert_precision, norm2, dot
    with pytest.raises(NarrowingOverflowError, match="index 1"):
        convert_precision(np.array([1.0, 1e39]), Precision.F32)
    out = convert_precision(np.array([np.inf, -np.inf, np.nan]), Precision.F32)
    assert np.isinf(out[0]) and np.isinf(out[1]) and np.isnan(out[2])
    assert convert_precision(np.array([1.0 + 2.0 ** -24]), Precision.F32)[0] == np.float32(1.0)
    assert norm2(np.array([3.0, 4.0])) == 5.0
    x = np.full(4, 1e20, dtype=np.float32)
    assert norm2(x) == pytest.approx(2e20, rel=1e-6)
    rng = np.random.default_rng(5)
    a, b = rng.standard_normal(100_000), rng.standard_normal(100_000)
    tiles = np.append(np.arange(0, a.size, 256), a.size)
    assert dot(a, b) == oracle.tree_dot(tiles, a, b)       # device order, bitwise
    assert dot(a, b) == pytest.approx(float(np.dot(a, b)), rel=1e-12)


def _solve_both(A, b, offs, pol, k, t, tol, oracle, stride=0, x0=None):
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
    pp = PrecisionPolicy.parse(pol)
    mp = build_mixed(A, pp, k=k, t=t, partition=BlockPartition(offs))
    rep = pcg_solve(A, b, mp, SolveConfig(res_tol=tol, record_true_residual_every=stride), x0=x0)
    orc = oracle.pcg_solve(A.row_ptr, A.col_idx, A.values, b, offs, kind=pp.kind.value,
                           adp_tol=pp.adp_tol, k=k, t=t, res_tol=tol, stride=stride,
                           order="device", x0=x0)
    return rep, orc


@pytest.mark.parametrize("pol", POLICIES)
def test_pcg_bitwise_vs_oracle_and_band_vs_reference(golden, cuda, oracle, pol):
    for name in golden_cases(golden):
        A = _matrix(golden, name)
        key = f"{name}/pcg/{pol}"
        tol, k, t = golden[f"{key}/meta"]
        rep, orc = _solve_both(A, golden[f"{name}/b"], golden[f"{name}/pcg/offsets"], pol,
                               int(k), int(t), float(tol), oracle, stride=5)
        # bit for bit against the device-order replay
        assert rep.iterations == orc["iterations"], name
        np.testing.assert_array_equal(rep.x, orc["x"], err_msg=name)
        np.testing.assert_array_equal([r.implicit_relres for r in rep.trace], orc["relres"])
        assert [r.branch for r in rep.trace] == orc["branch"]
        assert rep.final_true_relres == orc["final_true_relres"]
        tr = np.array([np.nan if r.true_relres is None else r.true_relres for r in rep.trace])
        np.testing.assert_array_equal(tr, orc["true_relres"])
        # within the band of the reference's own (sequential) run
        ref_it = int(golden[f"{key}/iterations"])
        assert abs(rep.iterations - ref_it) <= 2, (name, rep.iterations, ref_it)
        assert rep.converged


def test_pcg_x0_and_deterministic_rerun(cuda, oracle):
    from paper_2407_15973_b200 import problems
    cs = problems.make_config("c3", 16)
    offs = np.append(np.arange(0, cs.A.n, 64), cs.A.n)
    x0 = np.sin(np.arange(cs.A.n))
    rep1, orc = _solve_both(cs.A, cs.b, offs, "adaptive-lh:1e-6", 2, 2, 1e-10, oracle, x0=x0)
    rep2, _ = _solve_both(cs.A, cs.b, offs, "adaptive-lh:1e-6", 2, 2, 1e-10, oracle, x0=x0)
    np.testing.assert_array_equal(rep1.x, orc["x"])
    np.testing.assert_array_equal(rep1.x, rep2.x)
    assert rep1.iterations == rep2.iterations == orc["iterations"]


def test_pcg_error_paths(cuda):
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.solver import (BreakdownError, IndefiniteOperatorError,
                                              NonFiniteResidualError, SolveConfig, pcg_solve)
    U = PrecisionPolicy.parse("uniform")
    A = dense_to_csr(np.diag([1e308, 1e308]))
    with pytest.raises(BreakdownError):
        pcg_solve(A, np.array([1e-150, 1e-150]), build_mixed(A, U, nb=1, k=1, t=1))
    A = dense_to_csr(np.diag([1.0, -1.0]))
    with pytest.raises(IndefiniteOperatorError, match="preconditioner"):
        pcg_solve(A, np.array([0.0, 1.0]), build_mixed(A, U, nb=1, k=1, t=1))
    A = dense_to_csr([[1.0, 2.0], [2.0, 1.0]])
    with pytest.raises(IndefiniteOperatorError, match="matrix"):
        pcg_solve(A, np.array([1.0, -1.0]), build_mixed(A, U, nb=1, k=1, t=1))
    A = dense_to_csr([[1e-300]])
    with pytest.raises((NonFiniteResidualError, IndefiniteOperatorError)):
        pcg_solve(A, np.array([1e300]), build_mixed(A, U, nb=1, k=1, t=1))
    A = dense_to_csr(np.eye(3))
    rep = pcg_solve(A, np.zeros(3), build_mixed(A, U, nb=1))
    assert rep.converged and rep.iterations == 0 and rep.trace == []
    A = dense_to_csr(np.eye(6))
    rep = pcg_solve(A, np.arange(1.0, 7.0), build_mixed(A, U, nb=2))
    assert rep.converged and rep.iterations == 1
    np.testing.assert_array_equal(rep.x, np.arange(1.0, 7.0))
    assert rep.final_true_relres == 0.0 and rep.trace[0].true_relres == 0.0
    rng = np.random.default_rng(43)
    A = random_spd_csr(40, 0.25, rng)
    rep = pcg_solve(A, rng.standard_normal(40), build_mixed(A, U, nb=4), SolveConfig(max_iter=2))
    assert not rep.converged and rep.iterations == 2 and rep.final_true_relres > 0


def test_pcg_narrowing_overflow_raises(cuda):
    from paper_2407_15973_b200 import NarrowingOverflowError
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.solver import pcg_solve
    A = dense_to_csr(np.eye(4))
    mp = build_mixed(A, PrecisionPolicy.parse("fixed-low"), nb=2)
    with pytest.raises(NarrowingOverflowError, match="first at index 2"):
        pcg_solve(A, np.array([1.0, 2.0, 1e39, 1e39]), mp)


def test_tensor_io_stays_on_device(cuda):
    import torch
    from paper_2407_15973_b200 import problems
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.solver import pcg_solve
    cs = problems.make_config("c1", 16)
    mp = build_mixed(cs.A, PrecisionPolicy.parse("fixed-low"),
                     partition=BlockPartition.fixed_size(cs.A.n, 64))
    bt = torch.from_numpy(cs.b).cuda()
    rep = pcg_solve(cs.A, bt, mp)
    assert isinstance(rep.x, torch.Tensor) and rep.x.is_cuda
    rep2 = pcg_solve(cs.A, cs.b, mp)
    np.testing.assert_array_equal(rep.x.cpu().numpy(), rep2.x)


def test_unstaged_tiles_and_dense_rows_bitwise(cuda, oracle):
    """Tiles whose CSR slice exceeds the shared-memory stage fall back to
    direct global loads; results must not change."""
    from paper_2407_15973_b200 import Precision
    from paper_2407_15973_b200.bjac import BlockPartition, setup
    rng = np.random.default_rng(77)
    A = random_spd_csr(1200, 0.06, rng)          # ~140 nnz/row, tiles >> 8192 nnz
    r = rng.standard_normal(A.n)
    for offs in (np.arange(0, A.n + 1, 300), np.array([0, 5, 517, 1200]),
                 np.append(np.arange(0, A.n, 64), A.n)):
        part = BlockPartition(offs)
        d64, d32, v32, inb = oracle.setup_arrays(A.row_ptr, A.col_idx, A.values, offs)
        for k, t in ((1, 2), (2, 2), (3, 3)):
            z = setup(A, k=k, t=t, partition=part).apply(r)
            np.testing.assert_array_equal(
                z, oracle.bjac_apply(A.row_ptr, A.col_idx, A.values, inb, d64, k, t, r))
            z32 = setup(A, k=k, t=t, precision=Precision.F32, partition=part).apply(r.astype(np.float32))
            np.testing.assert_array_equal(
                z32, oracle.bjac_apply(A.row_ptr, A.col_idx, v32, inb, d32, k, t, r.astype(np.float32)))


@pytest.mark.parametrize("pol", ("fixed-low", "uniform", "adaptive-hl:1e-3"))
def test_pcg_many_tiles_per_cta_bitwise(cuda, oracle, pol):
    """n = 64 (512 tiles): every persistent CTA walks several tiles, so the
    shared-memory stage ring wraps around; still bit-identical."""
    from paper_2407_15973_b200 import problems
    cs = problems.make_config("c2", 64)
    offs = np.append(np.arange(0, cs.A.n, 64), cs.A.n)
    rep, orc = _solve_both(cs.A, cs.b, offs, pol, 2, 2, 1e-10, oracle)
    assert rep.iterations == orc["iterations"]
    np.testing.assert_array_equal(rep.x, orc["x"])
    np.testing.assert_array_equal([r.implicit_relres for r in rep.trace], orc["relres"])


@pytest.mark.parametrize("n,k,pol,tol", ((50, 2, "fixed-low", 1e-8), (50, 1, "uniform", 1e-8),
                                         (130, 2, "fixed-low", 1e-6), (130, 1, "uniform", 1e-6),
                                         (130, 2, "adaptive-lh:1e-4", 1e-6)))
def test_pcg_dot_sum_orders_bitwise(cuda, oracle, n, k, pol, tol):
    """n = 50: 489 tiles, the one-level sum in the kernels' final CTA.
    n = 130: 8,583 tiles > MPB_ONE_LEVEL_TILES, the two-level sum (33 full
    chunks and a ragged one) whose chunks the CTAs that claimed their last
    tiles sum while the kernels run.  k = 1 runs the unfused iteration (x/r
    update kernel), stride 3 and x0 the residual kernel."""
    from paper_2407_15973_b200 import problems
    cs = problems.make_config("c2", n)
    offs = np.append(np.arange(0, cs.A.n, 64), cs.A.n)
    x0 = np.cos(np.arange(cs.A.n) * 0.01)
    rep, orc = _solve_both(cs.A, cs.b, offs, pol, k, 2, tol, oracle, stride=3, x0=x0)
    assert rep.iterations == orc["iterations"]
    np.testing.assert_array_equal(rep.x, orc["x"])
    np.testing.assert_array_equal([r.implicit_relres for r in rep.trace], orc["relres"])
    tr = np.array([np.nan if r.true_relres is None else r.true_relres for r in rep.trace])
    np.testing.assert_array_equal(tr, orc["true_relres"])
    assert rep.final_true_relres == orc["final_true_relres"]


@pytest.mark.parametrize("pol", ("fixed-low", "adaptive-hl:1e-3"))
def test_slab_solver_single_rank_matches_single_gpu(cuda, oracle, pol):
    """The multi-GPU path (NCCL communicator, all-reduced scalar steps
    applied by k_apply_step) on one rank is bit-identical to pcg_solve."""
    from paper_2407_15973_b200 import problems
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.distributed import SlabSolver
    from paper_2407_15973_b200.policies import PrecisionPolicy
    from paper_2407_15973_b200.solver import SolveConfig
    cs = problems.make_config("c2", 16)
    offs = np.append(np.arange(0, cs.A.n, 64), cs.A.n)
    rep, orc = _solve_both(cs.A, cs.b, offs, pol, 2, 2, 1e-10, oracle, stride=4)
    ss = SlabSolver(cs.A, BlockPartition(offs), PrecisionPolicy.parse(pol), k=2, t=2, rank=0, nranks=1)
    drep = ss.solve(cs.b, SolveConfig(res_tol=1e-10, record_true_residual_every=4))
    assert drep.iterations == rep.iterations == orc["iterations"]
    np.testing.assert_array_equal(drep.x, orc["x"])
    np.testing.assert_array_equal([r.implicit_relres for r in drep.trace], orc["relres"])
    assert drep.final_true_relres == orc["final_true_relres"]


def test_row_patterns_and_generic_rows_bitwise(cuda, oracle):
    """Rows with a row pattern rebuild their columns from the pattern table;
    rows without one (too many distinct patterns, long rows) read SELL
    columns, mixed within the same tiles.  Both must be bit-identical."""
    from paper_2407_15973_b200 import Precision, problems
    from paper_2407_15973_b200.bjac import BlockPartition, setup
    cs = problems.make_config("c2", 16)
    P = setup(cs.A, k=2, t=2, partition=BlockPartition.fixed_size(cs.A.n, 64))
    info = P.plan.layout_info()
    assert (info["patterns"], info["generic_rows"]) == (27, 0)   # 7-point stencil, all boundary cases
    assert info["offset_slots"] == 7 and not info["offset_slot_update"]   # (+-16 is in-block at n = 16)
    rng = np.random.default_rng(91)
    A = random_spd_csr(3000, 0.0012, rng)                    # thousands of distinct patterns
    r = rng.standard_normal(A.n)
    for offs in (np.append(np.arange(0, A.n, 64), A.n), np.array([0, 7, 300, 301, 1500, 3000])):
        part = BlockPartition(offs)
        d64, d32, v32, inb = oracle.setup_arrays(A.row_ptr, A.col_idx, A.values, offs)
        for k, t in ((1, 1), (2, 2), (3, 3)):
            P64 = setup(A, k=k, t=t, partition=part)
            info = P64.plan.layout_info()
            assert info["patterns"] == 128
            assert P64.plan.large or 0 < info["generic_rows"] < A.n   # large blocks: no tiles
            np.testing.assert_array_equal(
                P64.apply(r), oracle.bjac_apply(A.row_ptr, A.col_idx, A.values, inb, d64, k, t, r))
            z32 = setup(A, k=k, t=t, precision=Precision.F32, partition=part).apply(r.astype(np.float32))
            np.testing.assert_array_equal(
                z32, oracle.bjac_apply(A.row_ptr, A.col_idx, v32, inb, d32, k, t, r.astype(np.float32)))
    b = rng.standard_normal(A.n)
    offs = np.append(np.arange(0, A.n, 64), A.n)
    for pol in ("fixed-low", "uniform"):
        rep, orc = _solve_both(A, b, offs, pol, 2, 2, 1e-10, oracle)
        assert rep.iterations == orc["iterations"]
        np.testing.assert_array_equal(rep.x, orc["x"])


def test_gpu_assembly_bitwise_vs_host(cuda):
    """The 7-point and 3-T operators and right-hand sides built on the GPU
    (mpb_assemble_stencil, mpb_expand_3t, mpb_splitmix64_uniform) equal the
    host generators bit for bit, boundary rows and weights included."""
    from paper_2407_15973_b200 import problems
    for name, n in (("c1", 12), ("c2", 16), ("c3", 24), ("c4", 8), ("c4", 3), ("c4", 2), ("c5", 20)):
        h = problems.make_config(name, n)
        d = problems.make_config(name, n, device=True)
        np.testing.assert_array_equal(d.A.row_ptr, h.A.row_ptr, err_msg=name)
        np.testing.assert_array_equal(d.A.col_idx, h.A.col_idx, err_msg=name)
        np.testing.assert_array_equal(d.A.values, h.A.values, err_msg=name)
        np.testing.assert_array_equal(d.b, h.b, err_msg=name)
    kap = np.exp(np.sin(np.arange(7 ** 3)))
    for wts in ((1.0, 1.0, 1.0), (1.0, 0.1, 0.1)):
        a = problems.diffusion_matrix(7, kap, wts)
        g = problems.diffusion_matrix(7, kap, wts, device=True)
        np.testing.assert_array_equal(g.values, a.values)
        np.testing.assert_array_equal(g.col_idx, a.col_idx)
    np.testing.assert_array_equal(problems.splitmix64_stream(12345, 1000, device=True),
                                  problems.splitmix64_stream(12345, 1000))


@pytest.mark.parametrize("pol", ("fixed-low", "uniform", "adaptive-hl:1e-3", "adaptive-lh:1e-4"))
def test_pcg_preconditioner_from_other_matrix(cuda, oracle, pol):
    """The outer SpMV and the true residuals multiply by the A passed to
    pcg_solve, the preconditioner keeps the values it was set up from
    (solver.py:154): solving A with build_mixed(diag_augment(A, p)) matches
    the oracle bit for bit, and the reference's run within the band."""
    import os
    from paper_2407_15973_b200 import SparseMatrix
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.problems import diag_augment
    from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "augment_golden.npz")
    with np.load(path) as z:
        g = {k: z[k] for k in z.files}
    for name in sorted({k.split("/")[0] for k in g}):
        rp, ci, v = (g[f"{name}/{s}"] for s in ("row_ptr", "col_idx", "values"))
        pd, k, t, tol = g[f"{name}/meta"]
        A = SparseMatrix(rp.size - 1, rp.size - 1, rp, ci, v)
        A2 = diag_augment(A, float(pd))
        offs, b = g[f"{name}/offsets"], g[f"{name}/b"]
        pp = PrecisionPolicy.parse(pol)
        mp = build_mixed(A2, pp, k=int(k), t=int(t), partition=BlockPartition(offs))
        cfg = SolveConfig(res_tol=float(tol), record_true_residual_every=4)
        for _ in range(2):   # also after A2's own solve (cached graph / values)
            rep = pcg_solve(A, b, mp, cfg)
            orc = oracle.pcg_solve(rp, ci, v, b, offs, kind=pp.kind.value, adp_tol=pp.adp_tol,
                                   k=int(k), t=int(t), res_tol=float(tol), stride=4,
                                   order="device", prec_values=A2.values)
            assert rep.iterations == orc["iterations"], name
            np.testing.assert_array_equal(rep.x, orc["x"], err_msg=name)
            np.testing.assert_array_equal([r.implicit_relres for r in rep.trace], orc["relres"])
            assert rep.final_true_relres == orc["final_true_relres"]
            assert abs(rep.iterations - int(g[f"{name}/{pol}/iterations"])) <= 2
            # the preconditioner's own matrix solves differently
            rep2 = pcg_solve(A2, b, mp, cfg)
            orc2 = oracle.pcg_solve(rp, ci, A2.values, b, offs, kind=pp.kind.value,
                                    adp_tol=pp.adp_tol, k=int(k), t=int(t), res_tol=float(tol),
                                    stride=4, order="device")
            np.testing.assert_array_equal(rep2.x, orc2["x"], err_msg=name)


@pytest.mark.parametrize("n,pol", ((64, "fixed-low"), (64, "uniform"), (64, "adaptive-hl:1e-3"),
                                   (32, "fixed-low"), (32, "adaptive-lh:1e-4"),
                                   (48, "fixed-low"), (48, "adaptive-hl:1e-3")))
def test_offset_slot_layout_bitwise(cuda, oracle, n, pol):
    """7-point stencil plans with 64-row blocks run the offset-slot kernels
    (k_bjac_dia, k_spmv_dia, k_update_first_dia: warp per block, no pattern
    lookups, masked absent slots).  n = 64: in-block entries at the diagonal
    and +-1 only (the fused update runs on the layout too); n = 32: +-32 is
    in-block as well (generic in-block mask).  Whole solves, bit for bit
    against the oracle, repeated (the tile sums are finished by whichever
    warp arrives last: any race there would show as a differing rerun), and
    with the preconditioner set up from another matrix of the same structure
    (the operator's own offset-slot values, mpb_csr.op_ib_val64)."""
    from paper_2407_15973_b200 import problems
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.problems import diag_augment
    from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
    cs = problems.make_config("c2", n)
    A = cs.A
    part = BlockPartition.fixed_size(A.n, 64)
    pp = PrecisionPolicy.parse(pol)
    mp = build_mixed(A, pp, k=2, t=3, partition=part)
    info = mp.any.plan.layout_info()
    assert info["offset_slots"] == 7 and info["generic_rows"] == 0
    assert info["offset_slot_update"] == (n >= 64)
    assert info["inblock_slots"] == (0b0011100 if n >= 64 else 0b0111110)
    cfg = SolveConfig(res_tol=1e-9, record_true_residual_every=5)
    kw = dict(kind=pp.kind.value, adp_tol=pp.adp_tol, k=2, t=3, res_tol=1e-9, stride=5, order="device")
    orc = oracle.pcg_solve(A.row_ptr, A.col_idx, A.values, cs.b, part.offsets, **kw)
    for _ in range(6):
        rep = pcg_solve(A, cs.b, mp, cfg)
        assert rep.iterations == orc["iterations"]
        np.testing.assert_array_equal(rep.x, orc["x"])
        np.testing.assert_array_equal([r.implicit_relres for r in rep.trace], orc["relres"])
        assert rep.final_true_relres == orc["final_true_relres"]
    # without strided true residuals a problem whose tiles' CTAs are all co-resident (n = 32: 128
    # tiles, one per SM; n = 48: 432 tiles, three per SM) runs the whole loop in one persistent
    # cooperative kernel (k_solve_small)
    for _ in range(3):
        rep = pcg_solve(A, cs.b, mp, SolveConfig(res_tol=1e-9))
        assert rep.iterations == orc["iterations"]
        np.testing.assert_array_equal(rep.x, orc["x"])
        np.testing.assert_array_equal([r.implicit_relres for r in rep.trace], orc["relres"])
        assert [r.branch for r in rep.trace] == list(orc["branch"])
        assert rep.final_true_relres == orc["final_true_relres"]
    A2 = diag_augment(A, 0.25)
    mp2 = build_mixed(A2, pp, k=2, t=3, partition=part)
    rep = pcg_solve(A, cs.b, mp2, SolveConfig(res_tol=1e-9))
    orc2 = oracle.pcg_solve(A.row_ptr, A.col_idx, A.values, cs.b, part.offsets, prec_values=A2.values, **kw)
    assert rep.iterations == orc2["iterations"]
    np.testing.assert_array_equal(rep.x, orc2["x"])
    rep = pcg_solve(A, cs.b, mp2, cfg)
    orc = oracle.pcg_solve(A.row_ptr, A.col_idx, A.values, cs.b, part.offsets, prec_values=A2.values, **kw)
    assert rep.iterations == orc["iterations"]
    np.testing.assert_array_equal(rep.x, orc["x"])
    assert rep.final_true_relres == orc["final_true_relres"]


def test_offset_slot_error_paths_both_solve_paths(cuda):
    """The reference's exceptions through the offset-slot kernels, on both
    solve paths of a small stencil problem (record_true_residual_every=0: the
    one persistent kernel; 3: the three-kernel graph iteration): narrowing
    overflow of the right-hand side (first index and count), a negative
    definite operator (indefinite preconditioner at iteration 1), the
    iteration cap, and a zero right-hand side."""
    from paper_2407_15973_b200 import NarrowingOverflowError, SparseMatrix, problems
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.solver import IndefiniteOperatorError, SolveConfig, pcg_solve
    cs = problems.make_config("c2", 20)
    A = cs.A
    part = BlockPartition.fixed_size(A.n, 64)
    low = build_mixed(A, PrecisionPolicy.parse("fixed-low"), k=2, t=2, partition=part)
    assert low.any.plan.layout_info()["offset_slots"] == 7
    b = cs.b.copy()
    b[[777, 4242]] = 1e39
    seen = []
    for stride in (0, 3):
        with pytest.raises(NarrowingOverflowError, match="first at index 777") as ei:
            pcg_solve(A, b, low, SolveConfig(record_true_residual_every=stride))
        seen.append(str(ei.value))
    assert seen[0] == seen[1]
    Aneg = SparseMatrix(A.n, A.m, A.row_ptr, A.col_idx, -A.values)
    for pol in ("uniform", "fixed-low"):
        mp = build_mixed(Aneg, PrecisionPolicy.parse(pol), k=2, t=2, partition=part)
        seen = []
        for stride in (0, 3):
            with pytest.raises(IndefiniteOperatorError, match="iteration 1: r'z") as ei:
                pcg_solve(Aneg, cs.b, mp, SolveConfig(record_true_residual_every=stride))
            seen.append(str(ei.value))
        assert seen[0] == seen[1]
    reps = [pcg_solve(A, cs.b, low, SolveConfig(max_iter=7, record_true_residual_every=s)) for s in (0, 3)]
    for rep in reps:
        assert not rep.converged and rep.iterations == 7
    np.testing.assert_array_equal(reps[0].x, reps[1].x)
    assert reps[0].final_true_relres == reps[1].final_true_relres
    assert reps[0].stats["kernel_launches"] < reps[1].stats["kernel_launches"]
    rep = pcg_solve(A, np.zeros(A.n), low)
    assert rep.converged and rep.iterations == 0
