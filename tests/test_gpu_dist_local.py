"""The multi-GPU solve (``mpb_pcg_solve_dist``: slab plans, ghost columns,
halo exchanges, all-reduced scalar steps, the fused distributed iteration)
run with 2 and 3 slab ranks on ONE GPU through the library's in-process
group (distributed.LocalSlabGroup, mpb_local_group_create): one host thread
per rank, one shared stream, halos as plain copies and the all-reduce as a
rank-ordered sum at host barriers -- no kernel waits on another rank.

Checked bit for bit against the CPU rank-split reference of
tests/test_distributed_gloo.py (global row kernels, dot products summed per
slab in device order and then over the slabs in rank order): x and the
whole implicit-residual trace.
"""
import numpy as np
import pytest

from test_distributed_gloo import _reference, _system

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("kind,adp_tol", [("fixed-low", None), ("adaptive-hl", 1e-3), ("uniform", None)])
def test_local_slab_group_matches_rank_split_reference(cuda, oracle, nranks, kind, adp_tol):
    from paper_2407_15973_b200.distributed import LocalSlabGroup
    from paper_2407_15973_b200.policies import PrecisionPolicy
    from paper_2407_15973_b200.solver import SolveConfig
    cs, part = _system()
    pol = PrecisionPolicy.parse(kind if adp_tol is None else f"{kind}:{adp_tol}")
    grp = LocalSlabGroup(cs.A, part, pol, nranks, k=cs.k, t=cs.t)
    assert all(s.ghosts > 0 for s in grp.slabs)
    x, reps = grp.solve(cs.b, SolveConfig(res_tol=cs.res_tol))
    x_ref, tr_ref = _reference(oracle, cs, part, nranks, pol.kind.value, pol.adp_tol)
    for rep in reps:  # every rank holds the same (global) trace
        assert rep.converged
        np.testing.assert_array_equal([t.implicit_relres for t in rep.trace], tr_ref)
    np.testing.assert_array_equal(x, x_ref)
    # a second solve reuses the ranks' buffers and gives the same bits
    x2, _ = grp.solve(cs.b, SolveConfig(res_tol=cs.res_tol))
    np.testing.assert_array_equal(x2, x)
    grp.close()


def test_local_slab_group_final_true_residual_and_x0(cuda, oracle):
    """Final true residual (halo of x + all-reduced norm) and a warm start
    through the slab path agree with the one-GPU solve to rounding of the
    dot order; the iteration count is within the band."""
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.distributed import LocalSlabGroup
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
    cs, part = _system("c3", 16)
    pol = PrecisionPolicy.parse("adaptive-lh:1e-6")
    cfg = SolveConfig(res_tol=cs.res_tol, record_true_residual_every=5)
    x0 = np.sin(np.arange(cs.A.n))
    grp = LocalSlabGroup(cs.A, part, pol, 2, k=cs.k, t=cs.t)
    x, reps = grp.solve(cs.b, cfg, x0=x0)
    one = pcg_solve(cs.A, cs.b, build_mixed(cs.A, pol, k=cs.k, t=cs.t,
                                            partition=BlockPartition(part.offsets)), cfg, x0=x0)
    assert abs(reps[0].iterations - one.iterations) <= 2
    assert reps[0].final_true_relres == reps[1].final_true_relres
    assert reps[0].final_true_relres == pytest.approx(one.final_true_relres, rel=1e-3)
    np.testing.assert_allclose(x, one.x, rtol=1e-8, atol=1e-12)
    grp.close()
