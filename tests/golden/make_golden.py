"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src, feeds
it matrices built by this repo's generators (bitwise identical to the
reference's own for the const/ani/dis/rand families; the config analogues
have no reference generator), and records what the reference's default
(numba) backend returns:

  * spmv / block_jacobi_sweeps outputs          (kernels_numba.py:37-70)
  * BjacPreconditioner.apply for fp64 and fp32   (bjac.py:127-149)
  * fmp_apply                                    (policies.py:154-160)
  * pcg_solve: iterations, trace, branches, x,
    final true relres per policy                 (solver.py:101-184)

The fixtures pin the CPU oracle (tests/test_oracle_golden.py) and, through
it, every GPU parity test.
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
import mpcg.problems  # noqa: E402
from mpcg import backend as ref_backend  # noqa: E402
from mpcg.bjac import BlockPartition as RefPartition, setup as ref_setup  # noqa: E402
from mpcg.policies import PrecisionPolicy as RefPolicy, build_mixed as ref_build, fmp_apply as ref_fmp  # noqa: E402
from mpcg.solver import SolveConfig as RefConfig, pcg_solve as ref_pcg  # noqa: E402

from paper_2407_15973_b200 import problems as P  # noqa: E402

assert ref_backend.name == "numba", "fixtures must come from the numba backend"

POLICIES = ("uniform", "fixed-low", "adaptive-hl:10", "adaptive-lh:1e-5",
            "adaptive-hl:1e-3")
KT = ((1, 1), (1, 2), (2, 2), (2, 3), (3, 2))


def rspd(n, density, seed):
    """Random symmetric diagonally dominant CSR (the reference's
    conftest.random_spd_csr recipe, pkg/tests/conftest.py:28-34)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, size=(n, n))
    a[rng.uniform(size=(n, n)) > density] = 0.0
    a = a + a.T
    np.fill_diagonal(a, np.abs(a).sum(axis=1) + 1.0)
    rows, cols = np.nonzero(a)
    return mpcg.SparseMatrix.from_coo(n, n, rows, cols, a[rows, cols])


def ref_matrix(M):
    return mpcg.SparseMatrix(M.n, M.m, M.row_ptr, M.col_idx, M.values)


def cases():
    out = {}
    out["rspd40"] = (rspd(40, 0.3, 31), np.random.default_rng(1).standard_normal(40),
                     [("nb8", RefPartition.equal_split(40, 8))])
    out["rspd200"] = (rspd(200, 0.05, 7), np.random.default_rng(2).standard_normal(200),
                      [("nb32", RefPartition.equal_split(200, 32)),
                       ("nb1", RefPartition.equal_split(200, 1))])
    fams = {"const8": (8, P.Family.CONST, 1.0, 0), "ani6": (6, P.Family.ANI, 100.0, 0),
            "dis10": (10, P.Family.DIS, 1000.0, 0), "rand12": (12, P.Family.RAND, 1000.0, 3)}
    from mpcg.problems import CoefficientField, Family as RefFamily, GridSpec, build_matrix
    for name, (n, fam, s, seed) in fams.items():
        # the reference's own assembly; this repo's generator must match it bitwise
        M = build_matrix(GridSpec(n), CoefficientField(RefFamily(fam.value), s, seed))
        mine = P.family_matrix(n, fam, s, seed)
        assert np.array_equal(M.values.view(np.uint64), mine.values.view(np.uint64))
        assert np.array_equal(M.col_idx, mine.col_idx) and np.array_equal(M.row_ptr, mine.row_ptr)
        N = n ** 3
        parts = [("nb32", RefPartition.equal_split(N, 32)),
                 ("r64", RefPartition(np.append(np.arange(0, N, 64), N)))]
        if N > 1024:
            parts.append(("nb2", RefPartition.equal_split(N, 2)))
        out[name] = (M, P.splitmix64_stream(100 + n, N) - 0.5, parts)
    for cname, n in (("c1", 16), ("c2", 16), ("c3", 16), ("c4", 6), ("c5", 16)):
        cs = P.make_config(cname, n)
        M = ref_matrix(cs.A)
        offs = np.append(np.arange(0, M.n, cs.block_rows), M.n)
        out[f"{cname}_n{n}"] = (M, cs.b, [(f"r{cs.block_rows}", RefPartition(offs))])
    return out


def main():
    fx = {}
    for name, (A, r, parts) in cases().items():
        fx[f"{name}/row_ptr"] = A.row_ptr
        fx[f"{name}/col_idx"] = A.col_idx
        fx[f"{name}/values"] = A.values
        fx[f"{name}/r"] = r
        x = np.cos(np.arange(A.n) * 0.37)
        fx[f"{name}/spmv64"] = mpcg.spmv(A, x)
        A32 = mpcg.convert_precision(A, mpcg.Precision.F32)
        fx[f"{name}/spmv32"] = mpcg.spmv(A32, x.astype(np.float32))
        for pname, part in parts:
            fx[f"{name}/{pname}/offsets"] = part.offsets
            for k, t in KT:
                for prec in (mpcg.Precision.F64, mpcg.Precision.F32):
                    pc = ref_setup(A, k=k, t=t, precision=prec, partition=part)
                    z = pc.apply(r.astype(prec.dtype))
                    fx[f"{name}/{pname}/apply_{prec}_k{k}t{t}"] = z
            mp = ref_build(A, RefPolicy.parse("fixed-low"), k=2, t=2, partition=part)
            fx[f"{name}/{pname}/fmp_k2t2"] = ref_fmp(mp, r)[0]
        # PCG on the first partition, every policy
        pname, part = parts[0]
        b = np.ones(A.n) if name.startswith(("const", "ani", "dis", "rand")) else \
            np.abs(r) + 0.1 if name.startswith("rspd") else r
        if name.startswith(("c1", "c2", "c3", "c4", "c5")):
            b = r
        fx[f"{name}/b"] = b
        fx[f"{name}/pcg/offsets"] = part.offsets
        tol = 1e-8 if name.startswith("c5") else 1e-10
        kk, tt = (2, 3) if name.startswith("c5") else (2, 2)
        for pol in POLICIES:
            mp = ref_build(A, RefPolicy.parse(pol), k=kk, t=tt, partition=part)
            rep = ref_pcg(A, b, mp, RefConfig(res_tol=tol, record_true_residual_every=5))
            key = f"{name}/pcg/{pol}"
            fx[f"{key}/iterations"] = np.int64(rep.iterations)
            fx[f"{key}/converged"] = np.int64(rep.converged)
            fx[f"{key}/relres"] = np.array([t_.implicit_relres for t_ in rep.trace])
            fx[f"{key}/true"] = np.array([np.nan if t_.true_relres is None else t_.true_relres
                                          for t_ in rep.trace])
            fx[f"{key}/branch"] = np.array([t_.branch == "low" for t_ in rep.trace], np.int8)
            fx[f"{key}/x"] = rep.x
            fx[f"{key}/final_true"] = np.float64(rep.final_true_relres)
            fx[f"{key}/meta"] = np.array([tol, kk, tt])
            print(f"{name:12s} {pol:18s} it={rep.iterations:4d} "
                  f"final_true={rep.final_true_relres:.3e}")
    # SplitMix64 / normal streams and the 3-T operator at a tiny size
    fx["streams/splitmix64_s7"] = mpcg.problems.splitmix64_stream(7, 64)
    fx["streams/splitmix64_s2pow40"] = mpcg.problems.splitmix64_stream(2 ** 40 + 3, 64)
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **fx)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
