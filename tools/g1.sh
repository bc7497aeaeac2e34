set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo "bench rc=$?"
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import time, numpy as np
from paper_2407_15973_b200 import problems
from paper_2407_15973_b200.bjac import BlockPartition
from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
cs = problems.make_config('c2', 128)
for pol in ('fixed-low','uniform'):
    mp = build_mixed(cs.A, PrecisionPolicy.parse(pol), nb=32, k=2, t=2)
    for rep in range(2):
        r = pcg_solve(cs.A, cs.b, mp, SolveConfig(res_tol=1e-10))
        print('nb32', pol, r.iterations, r.stats['device_seconds'], r.final_true_relres, flush=True)
" > gpurun_out/g1_nb32.log 2>&1; echo "nb32 rc=$?"
