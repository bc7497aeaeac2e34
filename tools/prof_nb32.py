"""Per-kernel times of one iteration on the reference's default nb=32
partition (Const n=128, b = ones): solver.profile_iteration."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2407_15973_b200 import problems
from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
from paper_2407_15973_b200.solver import SolveConfig, pcg_solve, profile_iteration
A = problems.family_matrix(128, problems.Family.CONST)
b = np.ones(A.n)
for pol in ("fixed-low", "uniform"):
    mp = build_mixed(A, PrecisionPolicy.parse(pol), nb=32)
    for _ in range(2):
        rep = pcg_solve(A, b, mp, SolveConfig(res_tol=1e-10))
    prof = profile_iteration(A, mp, config=SolveConfig(res_tol=1e-10), branch="low" if pol != "uniform" else "high", reps=10)
    print(json.dumps({"policy": pol, "iterations": rep.iterations, "solve_ms": rep.total_time * 1e3,
                      "us_per_iter": rep.total_time / rep.iterations * 1e6, "launches": rep.stats["kernel_launches"],
                      "profile_ms": {k: round(v, 4) for k, v in prof.items() if v}}), flush=True)
