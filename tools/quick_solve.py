import time, sys, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2407_15973_b200 import problems
from paper_2407_15973_b200.bjac import BlockPartition
from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
for name in sys.argv[1:] or ["c2"]:
    t0 = time.time(); cs = problems.make_config(name); t1 = time.time()
    part = BlockPartition.fixed_size(cs.A.n, cs.block_rows)
    for pol in cs.policies + ("uniform",):
        mp = build_mixed(cs.A, PrecisionPolicy.parse(pol), k=cs.k, t=cs.t, partition=part)
        for rep_i in range(3):
            torch.cuda.synchronize(); t2 = time.time()
            rep = pcg_solve(cs.A, cs.b, mp, SolveConfig(res_tol=cs.res_tol))
            t3 = time.time()
        print(f"{name} {pol}: gen {t1-t0:.1f}s it={rep.iterations} conv={rep.converged} true={rep.final_true_relres:.3e} "
              f"device {rep.total_time*1e3:.2f} ms ({rep.total_time/rep.iterations*1e6:.1f} us/it) wall {1e3*(t3-t2):.1f} ms launches={rep.stats['kernel_launches']}", flush=True)
