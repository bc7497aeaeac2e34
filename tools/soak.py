"""Rerun determinism soak: the same solves many times, every result compared
bit for bit with the first (x, trace, iteration count).  A race in the
lock-free pieces (streamed dot sums, arrival counters of the tile sums, grid
barriers of the small-problem kernel) would show as a differing rerun.

    python tools/soak.py [reps]
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2407_15973_b200 import problems
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    bad = 0
    for name, n, pol, stride in (("c2", 128, "fixed-low", 0), ("c2", 96, "adaptive-hl:1e-3", 0),
                                 ("c2", 64, "uniform", 7), ("c2", 48, "fixed-low", 0), ("c1", 32, "fixed-low", 0)):
        cs = problems.make_config(name, n, device=True)
        part = BlockPartition.fixed_size(cs.A.n, cs.block_rows)
        mp = build_mixed(cs.A, PrecisionPolicy.parse(pol), k=cs.k, t=cs.t, partition=part)
        b = cs.b if hasattr(cs.b, "cuda") and not isinstance(cs.b, np.ndarray) else torch.from_numpy(cs.b).cuda()
        cfg = SolveConfig(res_tol=cs.res_tol, record_true_residual_every=stride)
        ref = None
        for i in range(reps if n < 128 else max(reps // 2, 10)):
            rep = pcg_solve(cs.A, b, mp, cfg)
            key = (rep.iterations, hashlib.sha256(rep.x.cpu().numpy().tobytes()).hexdigest(),
                   tuple(r.implicit_relres for r in rep.trace), rep.final_true_relres)
            if ref is None:
                ref = key
            elif key != ref:
                bad += 1
                print(f"DIFFERENT rerun {i}: {name} n={n} {pol}: it {key[0]} vs {ref[0]}", flush=True)
        print(f"{name} n={n} {pol} stride={stride}: {ref[0]} iterations, launches {rep.stats['kernel_launches']}", flush=True)
    print(f"differing reruns: {bad}")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
