"""Fixtures for solves whose preconditioner was set up from ANOTHER matrix of
the same structure: pcg_solve(A, b, build_mixed(diag_augment(A, p), ...)).
The reference multiplies by the A it is given (pkg/src/mpcg/solver.py:154)
and preconditions with the augmented matrix's values.

Run in the build container (imports the reference read-only):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_augment_golden.py

Writes tests/golden/augment_golden.npz: per case the matrix, b, p_diag, and
per policy the reference's iterations, trace, branches, x and final true
relres.  Also checks this repo's problems.diag_augment against the
reference's bit for bit.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import mpcg  # noqa: E402  (the reference)
from mpcg import backend as ref_backend  # noqa: E402
from mpcg.bjac import BlockPartition as RefPartition  # noqa: E402
from mpcg.policies import PrecisionPolicy as RefPolicy, build_mixed as ref_build  # noqa: E402
from mpcg.problems import diag_augment as ref_augment  # noqa: E402
from mpcg.solver import SolveConfig as RefConfig, pcg_solve as ref_pcg  # noqa: E402

from paper_2407_15973_b200 import problems as P  # noqa: E402

assert ref_backend.name == "numba", "fixtures must come from the numba backend"

POLICIES = ("fixed-low", "uniform", "adaptive-hl:1e-3", "adaptive-lh:1e-4")


def main():
    fx = {}
    cases = (("c2_n16", "c2", 16, 1.0), ("c4_n6", "c4", 6, 0.5))
    for name, cfg, n, pd in cases:
        cs = P.make_config(cfg, n)
        A = mpcg.SparseMatrix(cs.A.n, cs.A.m, cs.A.row_ptr, cs.A.col_idx, cs.A.values)
        A2 = ref_augment(A, pd)
        mine = P.diag_augment(cs.A, pd)
        assert np.array_equal(A2.values.view(np.uint64), mine.values.view(np.uint64))
        offs = np.append(np.arange(0, A.n, cs.block_rows), A.n)
        part = RefPartition(offs)
        fx[f"{name}/row_ptr"] = A.row_ptr
        fx[f"{name}/col_idx"] = A.col_idx
        fx[f"{name}/values"] = A.values
        fx[f"{name}/prec_values"] = A2.values
        fx[f"{name}/offsets"] = offs
        fx[f"{name}/b"] = cs.b
        fx[f"{name}/meta"] = np.array([pd, cs.k, cs.t, cs.res_tol])
        for pol in POLICIES:
            mp = ref_build(A2, RefPolicy.parse(pol), k=cs.k, t=cs.t, partition=part)
            rep = ref_pcg(A, cs.b, mp, RefConfig(res_tol=cs.res_tol, record_true_residual_every=4))
            key = f"{name}/{pol}"
            fx[f"{key}/iterations"] = np.int64(rep.iterations)
            fx[f"{key}/relres"] = np.array([t.implicit_relres for t in rep.trace])
            fx[f"{key}/true"] = np.array([np.nan if t.true_relres is None else t.true_relres
                                          for t in rep.trace])
            fx[f"{key}/branch"] = np.array([t.branch == "low" for t in rep.trace], np.int8)
            fx[f"{key}/x"] = rep.x
            fx[f"{key}/final_true"] = np.float64(rep.final_true_relres)
            print(f"{name:8s} {pol:18s} it={rep.iterations:4d} final_true={rep.final_true_relres:.3e}")
    path = os.path.join(HERE, "augment_golden.npz")
    np.savez_compressed(path, **fx)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
