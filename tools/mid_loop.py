import sys, numpy as np, os
sys.path.insert(0, ".")
from paper_2407_15973_b200 import problems
from paper_2407_15973_b200.bjac import BlockPartition
from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
import torch
for n in (32, 52, 64, 96):
    cs = problems.make_config("c2", n)
    part = BlockPartition.fixed_size(cs.A.n, 64)
    mp = build_mixed(cs.A, PrecisionPolicy.parse("fixed-low"), k=2, t=2, partition=part)
    b = torch.from_numpy(cs.b).cuda()
    cfg = SolveConfig(res_tol=1e-10, record_true_residual_every=1000000)
    for _ in range(3): rep = pcg_solve(cs.A, b, mp, cfg)
    ds = [pcg_solve(cs.A, b, mp, cfg).stats["device_seconds"] for _ in range(10)]
    print(n, "RED", os.environ.get("MPB_RED"), rep.iterations, "loop us/iter", round(1e6 * float(np.median(ds)) / rep.iterations, 2), "tiles", mp.any.plan.ntiles)
