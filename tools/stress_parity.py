"""One-off parity sweep of the offset-slot kernels and the small-problem
kernel: C2-style systems on grids whose x-lines do not align with the 32-row
groups, all policy kinds, k and t from 1 to 4, with and without strided true
residuals (graph iteration vs one persistent kernel), each compared bit for
bit with the oracle's device-order replay.

    python tools/stress_parity.py [--quick]
"""
import itertools
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from oracle import oracle as O
    from paper_2407_15973_b200 import problems
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
    O.build()
    O.set_threads(os.cpu_count() or 1)
    quick = "--quick" in sys.argv
    grids = (16, 20, 28, 36, 44, 52, 68) if not quick else (20, 36)
    pols = ("fixed-low", "uniform", "adaptive-hl:1e-3", "adaptive-lh:1e-4")
    kts = ((1, 1), (1, 3), (2, 1), (2, 2), (2, 4), (3, 2), (3, 3)) if not quick else ((2, 2), (3, 3))
    bad = 0
    cases = 0
    t0 = time.time()
    for n in grids:
        cs = problems.make_config("c2", n)
        A = cs.A
        part = BlockPartition.fixed_size(A.n, 64)
        for pol, (k, t) in itertools.product(pols, kts):
            pp = PrecisionPolicy.parse(pol)
            mp = build_mixed(A, pp, k=k, t=t, partition=part)
            info = mp.any.plan.layout_info()
            for stride in (0, 3):
                kw = dict(kind=pp.kind.value, adp_tol=pp.adp_tol, k=k, t=t, res_tol=1e-9, stride=stride,
                          order="device", max_iter=400)
                orc = O.pcg_solve(A.row_ptr, A.col_idx, A.values, cs.b, part.offsets, **kw)
                rep = pcg_solve(A, cs.b, mp, SolveConfig(res_tol=1e-9, max_iter=400,
                                                         record_true_residual_every=stride))
                ok = (rep.iterations == orc["iterations"] and np.array_equal(rep.x, orc["x"])
                      and np.array_equal([r.implicit_relres for r in rep.trace], orc["relres"])
                      and [r.branch for r in rep.trace] == list(orc["branch"])
                      and rep.final_true_relres == orc["final_true_relres"])
                cases += 1
                if not ok:
                    bad += 1
                    print(f"MISMATCH n={n} {pol} k={k} t={t} stride={stride}: it {rep.iterations} vs "
                          f"{orc['iterations']}, launches {rep.stats['kernel_launches']}, layout {info}", flush=True)
        print(f"n={n}: N={A.n} tiles={mp.any.plan.ntiles} layout={info} ({time.time() - t0:.0f}s)", flush=True)
    # 3-T systems (96-row blocks, 81 patterns: the SELL + row-pattern kernels) and a 7-point grid
    # whose row count is not a multiple of 64 (no offset-slot layout): the same checks
    for name, n, rows in (("c4", 20, 96), ("c4", 28, 96), ("c2", 50, 64), ("c2", 30, 64)):
        cs = problems.make_config(name, n)
        A = cs.A
        part = BlockPartition.fixed_size(A.n, rows)
        for pol, (k, t) in itertools.product(pols, ((1, 2), (2, 2), (3, 1))):
            pp = PrecisionPolicy.parse(pol)
            mp = build_mixed(A, pp, k=k, t=t, partition=part)
            info = mp.any.plan.layout_info()
            for stride in (0, 4):
                kw = dict(kind=pp.kind.value, adp_tol=pp.adp_tol, k=k, t=t, res_tol=1e-9, stride=stride,
                          order="device", max_iter=300)
                orc = O.pcg_solve(A.row_ptr, A.col_idx, A.values, cs.b, part.offsets, **kw)
                rep = pcg_solve(A, cs.b, mp, SolveConfig(res_tol=1e-9, max_iter=300,
                                                         record_true_residual_every=stride))
                ok = (rep.iterations == orc["iterations"] and np.array_equal(rep.x, orc["x"])
                      and np.array_equal([r.implicit_relres for r in rep.trace], orc["relres"])
                      and [r.branch for r in rep.trace] == list(orc["branch"])
                      and rep.final_true_relres == orc["final_true_relres"])
                cases += 1
                if not ok:
                    bad += 1
                    print(f"MISMATCH {name} n={n} {pol} k={k} t={t} stride={stride}: it {rep.iterations} vs "
                          f"{orc['iterations']}, layout {info}", flush=True)
        print(f"{name} n={n}: N={A.n} tiles={mp.any.plan.ntiles} layout={info} ({time.time() - t0:.0f}s)", flush=True)
    print(f"{cases} cases, {bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
