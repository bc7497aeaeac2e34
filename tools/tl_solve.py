"""One config, one policy, a few solves on the device-resident problem (for
MPB_TIMELINE / MPB_VERBOSE diagnostics):  python tools/tl_solve.py c3 [policy] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_15973_b200 import problems  # noqa: E402
from paper_2407_15973_b200.bjac import BlockPartition  # noqa: E402
from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed  # noqa: E402
from paper_2407_15973_b200.solver import SolveConfig, pcg_solve  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cs = problems.make_config(name, device=True)
pol = sys.argv[2] if len(sys.argv) > 2 else cs.policies[0]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
mp = build_mixed(cs.A, PrecisionPolicy.parse(pol), k=cs.k, t=cs.t,
                 partition=BlockPartition.fixed_size(cs.A.n, cs.block_rows))
b = torch.as_tensor(cs.b).cuda()
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.time()
    rep = pcg_solve(cs.A, b, mp, SolveConfig(res_tol=cs.res_tol))
    t1 = time.time()
    print(f"{name} {pol}: it={rep.iterations} conv={rep.converged} true={rep.final_true_relres:.3e} "
          f"device {rep.total_time * 1e3:.2f} ms ({rep.total_time / rep.iterations * 1e6:.1f} us/it) "
          f"wall {1e3 * (t1 - t0):.1f} ms", flush=True)
