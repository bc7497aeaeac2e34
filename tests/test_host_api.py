"""Host-side logic of the drop-in API (no GPU): partitions, policies and the
branch rule, solver configuration and trace tooling, the sparse container,
problem generators (pinned bitwise to the reference's own assembly through
the golden fixtures) and the loud failure when no CUDA device is present.
Mirrors pkg/tests/test_bjac.py, test_policies.py, test_solver.py,
test_sparse.py and test_problems.py of the reference."""
import numpy as np
import pytest

from conftest import dense_to_csr


# ---- BlockPartition (pkg/tests/test_bjac.py:12-44) -------------------------

def test_partition_equal_split_and_ranges():
    from paper_2407_15973_b200.bjac import BlockPartition
    p = BlockPartition.equal_split(10, 3)
    np.testing.assert_array_equal(p.offsets, [0, 4, 7, 10])
    assert p.num_blocks == 3 and p.block_range(1) == (4, 7)
    np.testing.assert_array_equal(np.diff(BlockPartition.equal_split(9, 3).offsets), 3)
    np.testing.assert_array_equal(BlockPartition([0, 2, 5]).block_of_rows(), [0, 0, 1, 1, 1])
    np.testing.assert_array_equal(BlockPartition.fixed_size(10, 4).offsets, [0, 4, 8, 10])
    with pytest.raises(ValueError):
        BlockPartition.equal_split(3, 4)
    with pytest.raises(ValueError):
        BlockPartition.equal_split(3, 0)
    for bad in ([1, 3], [0, 2, 2], [0]):
        with pytest.raises(ValueError):
            BlockPartition(bad)
    with pytest.raises(IndexError):
        p.block_range(3)


# ---- policies (pkg/tests/test_policies.py:19-100) ---------------------------

def test_policy_parse_defaults_and_labels():
    from paper_2407_15973_b200.policies import PolicyKind, PrecisionPolicy
    assert PrecisionPolicy(PolicyKind.ADAPTIVE_HL).adp_tol == 10.0
    assert PrecisionPolicy(PolicyKind.ADAPTIVE_LH).adp_tol == 1e-5
    assert PrecisionPolicy.parse("adaptive-hl:0.5").adp_tol == 0.5
    assert PrecisionPolicy.parse("Uniform").kind is PolicyKind.UNIFORM
    assert PrecisionPolicy.parse("adaptive-lh:1e-5").label() == "adaptive-lh-1e-05"
    assert PrecisionPolicy.parse("adaptive-hl:10").label() == "adaptive-hl-10"
    with pytest.raises(ValueError, match="unknown policy"):
        PrecisionPolicy.parse("medium")
    with pytest.raises(ValueError, match="no adp_tol"):
        PrecisionPolicy.parse("uniform:3")
    with pytest.raises(ValueError, match="adp_tol"):
        PrecisionPolicy.parse("adaptive-hl:abc")
    with pytest.raises(ValueError):
        PrecisionPolicy(PolicyKind.ADAPTIVE_HL, adp_tol=0.0)
    assert not PrecisionPolicy(PolicyKind.UNIFORM).needs_low
    assert not PrecisionPolicy(PolicyKind.FIXED_LOW).needs_high


@pytest.mark.parametrize("kind,tol,relres,want", [
    ("UNIFORM", None, 1.0, "high"), ("FIXED_LOW", None, 1e-12, "low"),
    ("ADAPTIVE_HL", 1e-3, 1.0, "high"), ("ADAPTIVE_HL", 1e-3, 1e-3, "high"),
    ("ADAPTIVE_HL", 1e-3, 0.999e-3, "low"), ("ADAPTIVE_HL", 10.0, 1.0, "low"),
    ("ADAPTIVE_LH", 1e-3, 1.0, "low"), ("ADAPTIVE_LH", 1e-3, 1e-3, "low"),
    ("ADAPTIVE_LH", 1e-3, 0.999e-3, "high"), ("ADAPTIVE_LH", 10.0, 1.0, "high"),
    ("ADAPTIVE_HL", np.inf, 1.0, "low"), ("ADAPTIVE_HL", 5e-324, 1e-14, "high"),
    ("ADAPTIVE_LH", np.inf, 1.0, "high"), ("ADAPTIVE_LH", 5e-324, 1e-14, "low"),
])
def test_choose_branch_table(kind, tol, relres, want):
    from paper_2407_15973_b200.policies import PolicyKind, choose_branch
    assert choose_branch(PolicyKind[kind], tol, relres) == want


def test_choose_branch_rejects_bad_relres():
    from paper_2407_15973_b200.policies import PolicyKind, choose_branch
    for bad in (np.nan, -0.5, np.inf):
        with pytest.raises(ValueError):
            choose_branch(PolicyKind.ADAPTIVE_HL, 1.0, bad)
    with pytest.raises(ValueError, match="adp_tol"):
        choose_branch(PolicyKind.ADAPTIVE_HL, None, 1.0)


# ---- solver config and trace tooling (pkg/tests/test_solver.py) ------------

def test_solve_config():
    from paper_2407_15973_b200.solver import SolveConfig
    assert SolveConfig().res_tol == 1e-10
    assert SolveConfig().iteration_cap(100) == 1000
    assert SolveConfig().iteration_cap(5000) == 20000
    assert SolveConfig(max_iter=7).iteration_cap(10 ** 9) == 7
    for kw in ({"res_tol": 0.0}, {"max_iter": 0}, {"record_true_residual_every": -1}):
        with pytest.raises(ValueError):
            SolveConfig(**kw)


def test_detect_divergence_and_speedup():
    from paper_2407_15973_b200.solver import TINY, detect_divergence, speedup
    assert detect_divergence([1.0, 0.1, 0.01], [1.0, 0.1, 0.02]) is None
    assert detect_divergence([1.0, 0.5, 0.5, 0.5], [1.0, 0.1, 0.01, 0.001]) == 2
    assert detect_divergence([0.1], [0.01], delta_log10=1.0) is None
    assert detect_divergence([0.1], [0.009], delta_log10=1.0) == 1
    assert detect_divergence([0.0], [TINY]) is None
    assert detect_divergence([], [1.0]) is None

    class R:
        def __init__(self, t, c=True):
            self.total_time, self.converged = t, c
    assert speedup(R(3.0), R(2.0)) == 1.5
    with pytest.raises(ValueError):
        speedup(R(1.0, False), R(1.0))


def test_trace_csv_round_trip(tmp_path):
    from paper_2407_15973_b200.policies import PrecisionPolicy
    from paper_2407_15973_b200.solver import (IterationRecord, SolveReport, read_trace_csv,
                                              report_summary, trace_to_csv)
    trace = [IterationRecord(1, 0.5, None, "high", 0.1), IterationRecord(2, 1e-11, 2e-11, "low", 0.2)]
    rep = SolveReport(True, 2, trace, 2e-11, 0.2, PrecisionPolicy.parse("adaptive-hl:1"), None)
    p = tmp_path / "t.csv"
    trace_to_csv(rep, p)
    back = read_trace_csv(p)
    assert [(b.iteration, b.implicit_relres, b.true_relres, b.branch, b.wall_time) for b in back] == \
        [(1, 0.5, None, "high", 0.0), (2, 1e-11, 2e-11, "low", 0.0)]
    trace_to_csv(rep, p, include_timings=True)
    assert read_trace_csv(p)[1].wall_time == 0.2
    (tmp_path / "bad.csv").write_text("a,b\n1,2\n")
    with pytest.raises(ValueError, match="not a trace"):
        read_trace_csv(tmp_path / "bad.csv")
    d = report_summary(rep, extra={"n": 3})
    assert d["policy"] == "adaptive-hl-1" and d["iterations"] == 2 and d["n"] == 3


# ---- SparseMatrix (pkg/tests/test_sparse.py:32-100) -------------------------

def test_sparse_matrix_container():
    from paper_2407_15973_b200 import Precision, SparseMatrix
    A = SparseMatrix.from_coo(2, 2, [0, 0, 1, 0], [0, 1, 1, 0], [1.0, 2.0, 3.0, 4.0])
    assert A.nnz == 3
    np.testing.assert_array_equal(A.toarray(), [[5.0, 2.0], [0.0, 3.0]])
    B = SparseMatrix.from_coo(1, 4, [0, 0, 0], [3, 0, 2], [7.0, 1.0, 5.0])
    np.testing.assert_array_equal(B.col_idx, [0, 2, 3])
    C3 = SparseMatrix.from_coo(3, 3, [0, 1, 1, 2], [0, 0, 1, 0], [2.0, 5.0, -3.0, 7.0])
    np.testing.assert_array_equal(C3.diagonal(), [2.0, -3.0, 0.0])
    np.testing.assert_array_equal(C3.has_diagonal(), [True, True, False])
    assert A.precision is Precision.F64
    for bad in (([0, 2, 1], [0, 1], [1.0, 1.0]), ([1, 1, 2], [0, 1], [1.0, 1.0])):
        with pytest.raises(ValueError):
            SparseMatrix(2, 2, *bad)
    with pytest.raises(ValueError):
        SparseMatrix(1, 3, [0, 3], [0, 2, 1], [1.0, 1.0, 1.0])
    with pytest.raises(ValueError):
        SparseMatrix(1, 3, [0, 2], [1, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        SparseMatrix(1, 2, [0, 1], [2], [1.0])
    assert SparseMatrix(2, 3, [0, 2, 3], [1, 2, 0], [1.0, 2.0, 3.0]).nnz == 3


# ---- generators vs the reference's own assembly (golden fixtures) ----------

@pytest.mark.parametrize("name,n,fam,s,seed", [
    ("const8", 8, "CONST", 1.0, 0), ("ani6", 6, "ANI", 100.0, 0),
    ("dis10", 10, "DIS", 1000.0, 0), ("rand12", 12, "RAND", 1000.0, 3)])
def test_family_generators_bitwise(golden, name, n, fam, s, seed):
    from paper_2407_15973_b200 import problems as P
    A = P.family_matrix(n, P.Family[fam], s, seed)
    np.testing.assert_array_equal(A.row_ptr, golden[f"{name}/row_ptr"])
    np.testing.assert_array_equal(A.col_idx, golden[f"{name}/col_idx"])
    np.testing.assert_array_equal(A.values.view(np.uint64), golden[f"{name}/values"].view(np.uint64))


def test_splitmix64_matches_reference(golden):
    from paper_2407_15973_b200.problems import splitmix64_stream
    np.testing.assert_array_equal(splitmix64_stream(7, 64), golden["streams/splitmix64_s7"])
    np.testing.assert_array_equal(splitmix64_stream(2 ** 40 + 3, 64), golden["streams/splitmix64_s2pow40"])


def test_config_generators_shapes_and_symmetry(golden):
    from paper_2407_15973_b200 import problems as P
    c1 = P.make_config("c1")
    assert c1.A.n == 32768 and c1.A.nnz == 223232 and c1.block_rows == 64
    assert np.all(np.abs(c1.b) <= 1.0)
    for name, n in (("c2", 8), ("c3", 16), ("c5", 8)):
        cs = P.make_config(name, n)
        d = cs.A.toarray()
        assert np.array_equal(d, d.T)
        assert cs.A.nnz == 7 * n ** 3 - 6 * n ** 2
    c4 = P.make_config("c4", 5)
    d = c4.A.toarray()
    assert np.array_equal(d, d.T) and c4.A.n == 3 * 125
    assert c4.A.nnz == 3 * (7 * 125 - 6 * 25) + 4 * 125
    assert np.all(np.linalg.eigvalsh(d) > 0)
    # the config analogues in the fixtures were built by these generators
    for name, n in (("c1", 16), ("c2", 16), ("c3", 16), ("c5", 16), ("c4", 6)):
        cs = P.make_config(name, n)
        np.testing.assert_array_equal(cs.A.values, golden[f"{name}_n{n}/values"])
        np.testing.assert_array_equal(cs.b, golden[f"{name}_n{n}/b"])


# ---- no GPU: the product path fails loudly, never falls back ---------------

def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2407_15973_b200 import _lib, spmv
    A = dense_to_csr(np.eye(3))
    with pytest.raises(_lib.BackendUnavailableError):
        spmv(A, np.ones(3))
    from paper_2407_15973_b200.bjac import setup
    with pytest.raises(_lib.BackendUnavailableError):
        setup(A, nb=1)
