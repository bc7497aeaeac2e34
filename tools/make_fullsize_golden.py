"""Full-size oracle fixtures for the driver-run GPU suite
(tests/test_gpu_fullsize.py).

For each BASELINE config (C1-C5 at their full sizes) and policy, run the CPU
oracle (oracle/mpbjac_oracle.c, pinned bit for bit to the reference by
tests/test_oracle_golden.py) twice:

  * order="device": the GPU's tile-tree dot order.  The GPU solve must match
    it bit for bit: iteration count, implicit relres trace, branches, final
    true relres, and x (compared through its SHA-256 and a strided sample,
    since x itself is up to 1 GB);
  * order="sequential": the reference's own (numba, left-to-right) dot
    order.  The GPU's iteration count must lie within +-2 of it.

    python tools/make_fullsize_golden.py c2 [c4 ...] [--threads N]

Writes tests/golden/fullsize/<config>_<policy>.npz (a few KB to ~100 KB each).
The oracle is test infrastructure: this runs in the build container, and the
GPU box only reads the fixtures.
"""
import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "fullsize")

#: (config, policy) pairs with fixtures; C4 also runs aMP (hl:10, the
#: paper's default) and uniform
CASES = {
    "c1": ("uniform", "fixed-low"),
    "c2": ("fixed-low",),
    "c3": ("adaptive-lh:1e-6",),
    "c4": ("fixed-low", "adaptive-hl:10", "uniform"),
    "c5": ("fixed-low",),
    # the reference's own acceptance problems (pkg/tests/test_acceptance.py:
    # 226-274, pkg/test_output.txt:27-33): n=128, b = ones, its default
    # nb=32 partition (65,536-row blocks)
    "const128_nb32": ("uniform", "fixed-low"),
    "ani128_nb32": ("uniform", "fixed-low"),
}


class _System:
    def __init__(self, A, b, block_rows, k, t, res_tol, nb=None):
        self.A, self.b, self.block_rows, self.k, self.t, self.res_tol = A, b, block_rows, k, t, res_tol
        self.nb = nb


def make_system(cfg):
    """A BASELINE config, or one of the reference's acceptance problems."""
    from paper_2407_15973_b200 import problems
    if cfg.endswith("_nb32"):
        fam = problems.Family.CONST if cfg.startswith("const") else problems.Family.ANI
        s = 1.0 if fam is problems.Family.CONST else 1000.0
        A = problems.family_matrix(128, fam, s)
        return _System(A, np.ones(A.n), None, 2, 2, 1e-10, nb=32)
    cs = problems.make_config(cfg)
    return _System(cs.A, cs.b, cs.block_rows, cs.k, cs.t, cs.res_tol)


def partition_of(sysm):
    from paper_2407_15973_b200.bjac import BlockPartition
    if sysm.nb is not None:
        return BlockPartition.equal_split(sysm.A.n, sysm.nb)
    return BlockPartition.fixed_size(sysm.A.n, sysm.block_rows)


SAMPLES = 4096


def x_digest(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, np.float64).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--policy", default=None)
    ap.add_argument("--skip-sequential", action="store_true")
    args = ap.parse_args()
    from oracle import oracle as O
    from paper_2407_15973_b200.policies import PrecisionPolicy
    O.build()
    O.set_threads(args.threads)
    os.makedirs(OUT, exist_ok=True)
    for cfg in args.configs:
        t0 = time.time()
        cs = make_system(cfg)
        part = partition_of(cs)
        print(f"{cfg}: N={cs.A.n} nnz={cs.A.nnz} generated in {time.time() - t0:.0f}s", flush=True)
        for pol in ([args.policy] if args.policy else CASES[cfg]):
            pp = PrecisionPolicy.parse(pol)
            kw = dict(kind=pp.kind.value, adp_tol=pp.adp_tol, k=cs.k, t=cs.t, res_tol=cs.res_tol)
            t1 = time.time()
            dev = O.pcg_solve(cs.A.row_ptr, cs.A.col_idx, cs.A.values, cs.b, part.offsets,
                              order="device", **kw)
            t_dev = time.time() - t1
            fx = {
                "iterations": np.int64(dev["iterations"]),
                "converged": np.int64(dev["converged"]),
                "relres": dev["relres"],
                "branch": np.array([b == "low" for b in dev["branch"]], np.int8),
                "final_true": np.float64(dev["final_true_relres"]),
                "x_sha256": np.array(x_digest(dev["x"])),
                "x_sample_idx": np.linspace(0, cs.A.n - 1, SAMPLES).astype(np.int64),
                "meta": np.array([cs.A.n, cs.A.nnz, cs.k, cs.t, cs.res_tol, part.num_blocks]),
                "oracle_seconds_device": np.float64(t_dev),
                "oracle_threads": np.int64(args.threads),
            }
            fx["x_sample"] = dev["x"][fx["x_sample_idx"]]
            msg = f"  {pol:18s} device: it={dev['iterations']} true={dev['final_true_relres']:.4e} ({t_dev:.0f}s)"
            if not args.skip_sequential:
                t2 = time.time()
                seq = O.pcg_solve(cs.A.row_ptr, cs.A.col_idx, cs.A.values, cs.b, part.offsets,
                                  order="sequential", **kw)
                fx["seq_iterations"] = np.int64(seq["iterations"])
                fx["seq_final_true"] = np.float64(seq["final_true_relres"])
                fx["oracle_seconds_sequential"] = np.float64(time.time() - t2)
                msg += f"  sequential: it={seq['iterations']} true={seq['final_true_relres']:.4e}"
            path = os.path.join(OUT, f"{cfg}_{pol.replace(':', '_')}.npz")
            np.savez_compressed(path, **fx)
            print(msg, "->", os.path.relpath(path, ROOT), flush=True)
        del cs


if __name__ == "__main__":
    main()
