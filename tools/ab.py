"""A/B timing of the C2 solve under environment variants, interleaved:

    python tools/ab.py "" "MPB_NO_PDL=1" [--rounds 3] [--config c2] [--graph-iters 0]

Each variant runs in its own process (env is read at library load); prints
the median ms per solve of each variant over the rounds."""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
sys.path.insert(0, ROOT)
import torch
from paper_2407_15973_b200 import problems
from paper_2407_15973_b200.bjac import BlockPartition
from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
from paper_2407_15973_b200.solver import SolveConfig, pcg_solve
cs = problems.make_config(CFG, device=True)
mp = build_mixed(cs.A, PrecisionPolicy.parse(cs.policies[0]), k=cs.k, t=cs.t,
                 partition=BlockPartition.fixed_size(cs.A.n, cs.block_rows))
b = torch.from_numpy(cs.b).cuda()
cfg = SolveConfig(res_tol=cs.res_tol)
for _ in range(3): pcg_solve(cs.A, b, mp, cfg, graph_iters=G)
torch.cuda.synchronize()
out = []
for r in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): rep = pcg_solve(cs.A, b, mp, cfg, graph_iters=G)
    e1.record(); torch.cuda.synchronize()
    out.append(e0.elapsed_time(e1) / 5)
print(json.dumps({"ms": out, "iters": rep.iterations}))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--graph-iters", type=int, default=0)
    args = ap.parse_args()
    code = CHILD.replace("ROOT", repr(ROOT)).replace("CFG", repr(args.config)).replace("G)", f"{args.graph_iters})")
    res = {v: [] for v in args.variants}
    for _ in range(args.rounds):
        for v in args.variants:
            env = dict(os.environ)
            for kv in v.split():
                k, _, val = kv.partition("=")
                env[k] = val
            out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            line = [l for l in out.stdout.splitlines() if l.startswith("{")]
            if not line:
                print(f"[{v}] failed: {out.stderr[-500:]}")
                continue
            res[v] += json.loads(line[-1])["ms"]
    for v, ms in res.items():
        if ms:
            print(f"[{v or 'default'}] median {statistics.median(ms):.3f} ms  min {min(ms):.3f}  n={len(ms)}")


if __name__ == "__main__":
    main()
