"""Small solves that exercise every kernel family of the hot path, for
compute-sanitizer runs (tools/sanitize.sh): the fused single-GPU iteration
(warp-per-tile passes, TMA rings, PDL chaining, the device while loop), the
two-level chunk sums (forced with many tiles), the CTA-per-tile kernels of a
plan with generic rows, the large-block (nb=32-style) path, the standalone
apply / spmv / plugin kernels, and a 1-rank slab solve.

    python tools/sanitize_solve.py [--small]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2407_15973_b200 import kernels_b200 as K, problems
    from paper_2407_15973_b200.bjac import BlockPartition, setup
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
    from paper_2407_15973_b200.sparse import Precision, SparseMatrix
    out = []
    for name, n in (("c2", 16), ("c4", 6), ("c3", 16)):
        cs = problems.make_config(name, n)
        part = BlockPartition.fixed_size(cs.A.n, cs.block_rows)
        for pol in ("fixed-low", "uniform", "adaptive-hl:1e-3"):
            mp = build_mixed(cs.A, PrecisionPolicy.parse(pol), k=cs.k, t=cs.t, partition=part)
            rep = pcg_solve(cs.A, cs.b, mp, SolveConfig(res_tol=cs.res_tol, max_iter=40,
                                                         record_true_residual_every=7))
            out.append((name, pol, rep.iterations))
    # many tiles: the two-level (chunked) sums and chunk owners (> 8192 tiles)
    cs = problems.make_config("c2", 136)
    mp = build_mixed(cs.A, PrecisionPolicy.parse("fixed-low"), k=2, t=2,
                     partition=BlockPartition.fixed_size(cs.A.n, 64))
    rep = pcg_solve(cs.A, cs.b, mp, SolveConfig(res_tol=1e-10, max_iter=6))
    out.append(("c2_136", "fixed-low", rep.iterations))
    # large blocks (the reference's default nb=32 partition)
    A = problems.family_matrix(16, problems.Family.CONST)
    for pol in ("uniform", "fixed-low"):
        rep = pcg_solve(A, np.ones(A.n), build_mixed(A, PrecisionPolicy.parse(pol), nb=4),
                        SolveConfig(res_tol=1e-10, max_iter=20))
        out.append(("const16_nb4", pol, rep.iterations))
    # generic rows (no row pattern): a random SPD matrix
    rng = np.random.default_rng(5)
    a = rng.uniform(-1, 1, (300, 300))
    a[rng.uniform(size=a.shape) > 0.05] = 0
    a = a + a.T
    np.fill_diagonal(a, np.abs(a).sum(1) + 1)
    r_, c_ = np.nonzero(a)
    R = SparseMatrix.from_coo(300, 300, r_, c_, a[r_, c_])
    for pol in ("uniform", "fixed-low"):
        rep = pcg_solve(R, np.ones(300), build_mixed(R, PrecisionPolicy.parse(pol), nb=30),
                        SolveConfig(res_tol=1e-10))
        out.append(("rspd300", pol, rep.iterations))
    # standalone apply / plugin kernels
    P = setup(R, nb=30, k=3, t=2, precision=Precision.F32)
    P.apply(np.ones(300, np.float32))
    y, tmp = np.zeros(300), np.zeros(300)
    rows = np.repeat(np.arange(300), np.diff(R.row_ptr))
    K.block_jacobi_sweeps(R.row_ptr, R.col_idx, R.values, rows == R.col_idx, np.diag(a), 3,
                          np.ones(300), y, tmp, 10, 290)
    o = np.empty(300)
    K.csr_matvec(R.row_ptr, R.col_idx, R.values, np.ones(300), o)
    K.dot_seq(o, o)
    for row in out:
        print(*row)


if __name__ == "__main__":
    main()
