import sys, numpy as np
sys.path.insert(0, '.')
from paper_2407_15973_b200 import problems
from paper_2407_15973_b200.bjac import BlockPartition
from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
import torch
cs = problems.make_config("c1", device=True)
part = BlockPartition.fixed_size(cs.A.n, 64)
for pol in ("fixed-low", "uniform"):
    mp = build_mixed(cs.A, PrecisionPolicy.parse(pol), k=2, t=2, partition=part)
    b = torch.from_numpy(cs.b).cuda() if isinstance(cs.b, np.ndarray) else cs.b
    for _ in range(3): rep = pcg_solve(cs.A, b, mp, SolveConfig(res_tol=1e-10))
    ds = [pcg_solve(cs.A, b, mp, SolveConfig(res_tol=1e-10)).stats["device_seconds"] for _ in range(10)]
    print(pol, rep.iterations, "loop us/iter", 1e6 * float(np.median(ds)) / rep.iterations, "launches", rep.stats["kernel_launches"])
