"""Full-size parity: the GPU solve of a BASELINE config against the oracle's
device-order replay (all host cores), bit for bit: iteration count, implicit
relres trace, branch trace and x.  Prints one JSON line.

    python tools/fullsize_parity.py c2 [--threads 16] [--policy fixed-low]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--policy", default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--max-iter", type=int, default=None, help="cap both solves (C5: hours on the CPU)")
    args = ap.parse_args()
    from oracle import oracle as O
    from paper_2407_15973_b200 import problems
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
    t0 = time.time()
    cs = problems.make_config(args.config, args.n)
    policy = args.policy or cs.policies[0]
    part = BlockPartition.fixed_size(cs.A.n, cs.block_rows)
    pp = PrecisionPolicy.parse(policy)
    t_build = time.time() - t0
    mp = build_mixed(cs.A, pp, k=cs.k, t=cs.t, partition=part)
    rep = pcg_solve(cs.A, cs.b, mp, SolveConfig(res_tol=cs.res_tol, max_iter=args.max_iter))
    O.build()
    O.set_threads(args.threads)
    t1 = time.time()
    orc = O.pcg_solve(cs.A.row_ptr, cs.A.col_idx, cs.A.values, cs.b, part.offsets, kind=pp.kind.value,
                      adp_tol=pp.adp_tol, k=cs.k, t=cs.t, res_tol=cs.res_tol, order="device",
                      max_iter=args.max_iter)
    t_orc = time.time() - t1
    rel = np.array([r.implicit_relres for r in rep.trace])
    same_trace = rel.size == orc["relres"].size and bool(np.array_equal(rel, orc["relres"]))
    out = {
        "config": args.config, "n": cs.n, "rows": cs.A.n, "nnz": cs.A.nnz, "policy": policy,
        "gpu_iterations": rep.iterations, "oracle_iterations": orc["iterations"],
        "trace_bitwise": same_trace,
        "branches_equal": [r.branch for r in rep.trace] == orc["branch"],
        "x_bitwise": bool(np.array_equal(rep.x, orc["x"])),
        "x_max_abs_diff": float(np.max(np.abs(rep.x - orc["x"]))),
        "gpu_final_true_relres": rep.final_true_relres,
        "oracle_final_true_relres": orc["final_true_relres"],
        "converged": rep.converged, "max_iter": args.max_iter, "oracle_threads": args.threads,
        "oracle_seconds": round(t_orc, 1), "build_seconds": round(t_build, 1),
    }
    print(json.dumps(out), flush=True)
    return 0 if (out["trace_bitwise"] and out["x_bitwise"]) else 1


if __name__ == "__main__":
    sys.exit(main())
