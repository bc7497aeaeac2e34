#!/usr/bin/env python
"""Benchmark: PCG time-to-solution of the mixed-precision BJAC-PCG hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
                    [--policy fixed-low] [--impl b200|reference]

One step = one complete ``pcg_solve`` to rtol (default: BASELINE.json
configs[1] = C2, 128^3 lognormal diffusion, fixed-low fMP-BJAC, 64-row
blocks, k = t = 2, rtol 1e-10).  ``value`` is whole-job solves per second
with b already resident in HBM (device-timed with CUDA events, max over
ranks); ``e2e`` is the same through the public API with pinned host b and a
host read of x every step.  The line also carries the per-kernel roofline
(live CUDA-event timings of each kernel of an iteration, algorithmic bytes
of DESIGN.md §4), the CPU baseline (the oracle restatement of the
reference, 1 thread, bounded sample), clocks sampled during the timed
region and the number of kernels launched.

With --gpus N under torchrun the one system is cut into z-slabs, one per
rank (strong scaling: ``value`` stays global solves per second), with NCCL
halos and all-reduces inside the iteration graph;
``--impl reference`` times the reference's CPU
implementation (the oracle port, all host threads) on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

def ref_iterations(cfg: str, policy: str):
    """Iterations of the reference-order (sequential dot) solve to rtol,
    from the oracle fixtures of tools/make_fullsize_golden.py; None when no
    fixture exists for this (config, policy)."""
    path = os.path.join(ROOT, "tests", "golden", "fullsize", f"{cfg}_{policy.replace(':', '_')}.npz")
    if not os.path.exists(path):
        return None
    with np.load(path) as z:
        return int(z["seq_iterations"]) if "seq_iterations" in z.files else None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--policy", default=None)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--cpu-iters", type=int, default=40,
                    help="iterations of the bounded CPU-baseline sample")
    ap.add_argument("--ref-budget", type=float, default=40.0,
                    help="--impl reference: seconds a whole solve may take before steps "
                         "become capped samples extrapolated to the known iteration count")
    ap.add_argument("--ref-iters", type=int, default=60,
                    help="--impl reference: iterations of a capped sample step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU slab path even at N=1 (always on for N>1)")
    ap.add_argument("--profile-reps", type=int, default=20)
    ap.add_argument("--profile-only", action="store_true",
                    help="one solve, then only the per-kernel launches (for ncu: graph-node "
                         "kernels of the solve are not replayed by ncu)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(busy)) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def kernel_bytes(Z, N, branch, ntiles, Zb):
    """Algorithmic bytes per launch, SURVEY.md §8(d) model (CSR, int32
    row_ptr and col_idx, every array streamed once, gathered vector entries
    counted once): what ``roofline.achieved`` is computed from."""
    if branch == "low":
        first, mid, last, pupd = 8 * Z + 16 * N, 8 * Z + 20 * N, 8 * Z + 24 * N, 24 * N
    else:
        first, mid, last, pupd = 12 * Z + 20 * N, 12 * Z + 28 * N, 12 * Z + 28 * N, 24 * N
    # fused x/r update + next first pass: both, r read once
    return {"bjac_first": first, "bjac_middle": mid, "bjac_last": last,
            "pupdate": pupd, "spmv_pq": 12 * Z + 20 * N, "update": 48 * N,
            "update_first": 48 * N + first - 8 * N, "scalar": 8 * ntiles,
            # fused mode: p = z + beta p rebuilt inside the SpMV (p read once)
            "spmv_p": 12 * Z + 20 * N + pupd - 8 * N,
            # wave kernel: fused update + first pass + the next last pass
            # (the last pass's r and z1 come from the same kernel)
            "wave": 48 * N + first - 8 * N + last - 8 * N - (4 if branch == "low" else 8) * N}


def format_bytes(Z, N, branch, Zb):
    """Bytes our layout has to move per launch: SELL values
    only (row-pattern rows carry no column index), 2-byte row metadata, the
    first pass reads in-block entries only (Zb), z_in / p gathered once."""
    if branch == "low":
        first, mid, last, pupd = 4 * Zb + 14 * N, 4 * Z + 18 * N, 4 * Z + 18 * N, 20 * N
    else:
        first, mid, last, pupd = 8 * Zb + 18 * N, 8 * Z + 26 * N, 8 * Z + 26 * N, 24 * N
    return {"bjac_first": first, "bjac_middle": mid, "bjac_last": last,
            "pupdate": pupd, "spmv_pq": 8 * Z + 18 * N, "update": 48 * N,
            "update_first": 48 * N + first - 8 * N,
            "spmv_p": 8 * Z + 18 * N + pupd - 8 * N,
            "wave": 48 * N + first - 8 * N + last - 8 * N - (4 if branch == "low" else 8) * N}


def inblock_nnz(A, part):
    """Stored entries whose column lies in the row's own block (Zb)."""
    blk = part.block_of_rows()
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    return int(np.count_nonzero(blk[rows] == blk[A.col_idx]))


def cpu_sample(cs, part, policy, iters, threads, order="sequential"):
    """Oracle solve capped at `iters` iterations; returns seconds."""
    from oracle import oracle as O
    O.build()
    O.set_threads(threads)
    kind, _, tol = policy.partition(":")
    t0 = time.perf_counter()
    out = O.pcg_solve(cs.A.row_ptr, cs.A.col_idx, cs.A.values, cs.b, part.offsets,
                      kind=kind, adp_tol=float(tol) if tol else None, k=cs.k, t=cs.t,
                      res_tol=cs.res_tol, max_iter=iters, order=order)
    dt = time.perf_counter() - t0
    return dt, out["iterations"]


def metric_name(cfg):
    return (f"PCG solves/s to rtol {cfg.res_tol:g} (time-to-solution), "
            f"{cfg.name.upper()} {cfg.n}^3")


def config_dict(cs, part, policy, extra=None):
    d = {"workload": f"{cs.name.upper()}: {cs.note}, n={cs.n} (N={cs.A.n}, nnz={cs.A.nnz}), "
                     f"{cs.block_rows}-row BJAC blocks, policy {policy}, k={cs.k} t={cs.t}, "
                     f"rtol {cs.res_tol:g}, x0=0",
         "n_rows": cs.A.n, "nnz": cs.A.nnz, "blocks": part.num_blocks,
         "policy": policy, "k": cs.k, "t": cs.t, "res_tol": cs.res_tol,
         "l2": "inputs larger than L2 (>= 650 MB streamed per iteration vs 126 MB L2); no flush"}
    if extra:
        d.update(extra)
    return d


def run_reference(args, world, rank):
    """The reference's CPU implementation of the path (the oracle port of
    kernels_numba.py / bjac.py / solver.py, reference dot order, all host
    threads) on rank 0.  A step is one whole solve to rtol when that fits
    --ref-budget seconds (C1, C2 on a 16-core host); otherwise a capped
    sample scaled by the reference-order iteration count of the oracle
    fixtures -- and no line at all (an "unavailable" line) when that count is
    unknown."""
    from paper_2407_15973_b200 import problems
    from paper_2407_15973_b200.bjac import BlockPartition
    if rank != 0:
        return
    cs = problems.make_config(args.config)
    policy = args.policy or cs.policies[0]
    part = BlockPartition.fixed_size(cs.A.n, cs.block_rows)
    threads = os.cpu_count() or 1
    it_full = ref_iterations(cs.name, policy)
    # probe: a short capped solve gives the per-iteration cost
    dt, its = cpu_sample(cs, part, policy, 10, threads)
    est = dt / max(its, 1) * (it_full or 10 ** 9)
    whole = est <= args.ref_budget
    if not whole and it_full is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"no reference-order iteration count for {cs.name}/{policy} and a whole "
                          f"solve exceeds the {args.ref_budget:g} s budget"}), flush=True)
        return
    cap = None if whole else args.ref_iters
    for _ in range(args.warmup):   # warm-up: short capped solves (page cache, thread pool)
        cpu_sample(cs, part, policy, 10, threads)
    times, iters = [], []
    for _ in range(args.steps):
        dt, its = cpu_sample(cs, part, policy, cap, threads)
        times.append(dt)
        iters.append(its)
    if whole:
        step_s = float(np.mean(times))
        solve_s = step_s
        sample = (f"{cs.name.upper()}: whole solves to rtol {cs.res_tol:g} ({iters[0]} iterations; "
                  f"oracle restatement of the reference, reference dot order, {threads} OpenMP threads)")
    else:
        step_s = float(np.mean(times))
        solve_s = float(np.mean([t / i for t, i in zip(times, iters)])) * it_full
        sample = (f"{cs.name.upper()} solve capped at {args.ref_iters} iterations per step "
                  f"(oracle restatement of the reference, reference dot order, {threads} OpenMP "
                  f"threads), scaled to the {it_full}-iteration reference-order solve "
                  f"(tests/golden/fullsize); ms_per_step is the solve time, step_s the sample")
    value = 1.0 / solve_s
    line = {"impl": "reference", "metric": metric_name(cs), "value": value,
            "unit": "solve/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * solve_s,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64 CG / f32 preconditioner", "data": "synthetic (seeded SplitMix64)",
            "config": config_dict(cs, part, policy, {"parallelism": "1 CPU process"}),
            "iterations": iters[0] if whole else it_full, "whole_solves": whole,
            "step_s": step_s,
            "cpu_baseline": {"value": value, "unit": "solve/s", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "solve/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _inblock_nnz_local(row_ptr, col_idx, offsets, m):
    """Zb of a slab (ghost columns >= m are never in a block)."""
    blk = np.searchsorted(offsets, np.arange(m), side="right") - 1
    rows = np.repeat(np.arange(m), np.diff(row_ptr))
    c = np.asarray(col_idx, np.int64)
    own = c < m
    return int(np.count_nonzero(blk[rows[own]] == blk[c[own]]))


def run_b200(args, world, rank, local):
    import torch
    from paper_2407_15973_b200 import _lib, problems
    from paper_2407_15973_b200.bjac import BlockPartition
    from paper_2407_15973_b200.policies import PrecisionPolicy, build_mixed
    from paper_2407_15973_b200.solver import SolveConfig, pcg_solve, profile_iteration

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cs = problems.make_config(args.config, device=True)   # GPU-side assembly (bit-identical)
    policy = args.policy or cs.policies[0]
    part = BlockPartition.fixed_size(cs.A.n, cs.block_rows)
    pp = PrecisionPolicy.parse(policy)
    cfg = SolveConfig(res_tol=cs.res_tol)
    sharded = world > 1 or args.sharded
    if sharded:
        # strong scaling: one global solve, z-slabs over the ranks
        from paper_2407_15973_b200.distributed import SlabSolver
        ss = SlabSolver(cs.A, part, pp, k=cs.k, t=cs.t, rank=rank, nranks=world, device=local)
        lo, hi = ss.slab.lo, ss.slab.hi

        def solve(b):
            return ss.solve(b, cfg)

        def profile(branch):
            return ss.profile_iteration(cfg, branch=branch, reps=args.profile_reps)
        A_loc, plan = ss.A_loc, ss.mp.any.plan
        zb = _inblock_nnz_local(ss.slab.row_ptr, ss.slab.col_idx, ss.slab.offsets, hi - lo)
    else:
        mp = build_mixed(cs.A, pp, k=cs.k, t=cs.t, partition=part)
        lo, hi = 0, cs.A.n

        def solve(b):
            return pcg_solve(cs.A, b, mp, cfg)

        def profile(branch):
            return profile_iteration(cs.A, mp, config=cfg, branch=branch, reps=args.profile_reps)
        A_loc, plan = cs.A, mp.any.plan
        zb = inblock_nnz(cs.A, part)
    m = hi - lo
    b_loc = np.ascontiguousarray(cs.b[lo:hi])
    b_dev = torch.from_numpy(b_loc).cuda()

    for _ in range(max(args.warmup, 1)):
        rep = solve(b_dev)
    if args.profile_only:
        branch = rep.trace[-1].branch if rep.trace else "low"
        print(json.dumps({"profile_iteration_ms": profile(branch)}), flush=True)
        return
    # ---- device-resident timed region --------------------------------------
    sampler = ClockSampler(local)
    sampler.start()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    iters = []
    ev0.record()
    for _ in range(args.steps):
        rep = solve(b_dev)
        launches += rep.stats["kernel_launches"]
        iters.append(rep.iterations)
    ev1.record()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = args.steps / (ms / 1e3)        # global solves per second

    # ---- end to end through the public API, host buffers -------------------
    b_pin = torch.from_numpy(b_loc).pin_memory()
    x_pin = torch.empty(m, dtype=torch.float64).pin_memory()
    for _ in range(max(args.warmup, 1)):   # warm-up through the same path (first-use costs)
        x_pin.copy_(solve(b_pin).x, non_blocking=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    d2h = 0
    for _ in range(args.steps):
        r2 = solve(b_pin)
        x_pin.copy_(r2.x, non_blocking=True)
        d2h += 8 * m + r2.iterations * (3 * 8 + 4)
    e1.record()
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ems], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    e2e = {"value": args.steps / (ems / 1e3), "unit": "solve/s",
           "h2d_bytes_per_step": 8 * m, "d2h_bytes_per_step": d2h // args.steps,
           "ms_per_step": ems / args.steps,
           "note": "per rank: its slab of b in, its slab of x and the trace out" if sharded else
                   "b in, x and the trace out"}

    # ---- per-kernel roofline (live CUDA events on the solve stream) --------
    branch = rep.trace[-1].branch if rep.trace else "low"
    prof = profile(branch)
    ntiles = plan.ntiles
    kb = kernel_bytes(A_loc.nnz, m, branch, ntiles, zb)
    fb = format_bytes(A_loc.nnz, m, branch, zb)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except OSError:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    kernels = {}
    fused = prof.get("update_first", 0.0) > 0
    wave = prof.get("wave", 0.0) > 0
    if wave:    # what the solve runs: SpMV with the p rebuild, wave (x/r update + first pass + next last pass)
        prof = dict(prof, spmv_p=prof["spmv_pq"])
        run = ("spmv_p", "wave")
    elif fused:   # what the solve runs: last pass, SpMV with the p rebuild, x/r update + next first pass
        prof = dict(prof, spmv_p=prof["spmv_pq"])
        run = ("bjac_last", "spmv_p", "update_first")
    else:
        run = ("bjac_first", "bjac_last", "pupdate", "spmv_pq", "update")
    for name in run:
        # per-launch time with the launches chained by programmatic dependent
        # launch, as the solve graph runs them; the cold single launch (launch
        # latency, ramp and drain between two events) is reported beside it
        base = "spmv_pq" if name == "spmv_p" else name
        t_ms = prof.get(base + "_chained", 0.0) or prof[name]
        t_cold = prof[name]
        if t_ms <= 0:
            continue
        gbs = kb[name] / (t_ms * 1e-3) / 1e9
        fgbs = fb[name] / (t_ms * 1e-3) / 1e9
        kernels[name] = {"ms": round(t_ms, 5), "bytes": kb[name], "gbs": round(gbs, 1),
                         "frac": round(gbs / peak, 4), "format_bytes": fb[name],
                         "format_gbs": round(fgbs, 1), "format_frac": round(fgbs / peak, 4),
                         "ms_cold": round(t_cold, 5),
                         "frac_cold": round(kb[name] / (t_cold * 1e-3) / 1e9 / peak, 4)}
    per_iter_share = {k: v["ms"] for k, v in kernels.items()}
    dom = max(kernels, key=lambda k: per_iter_share[k])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and world == 1:
        with open(tpath) as fh:
            tj = json.load(fh).get(cs.name, {})
            traffic = tj.get({"spmv_p": "spmv_pq"}.get(dom, dom))
    t_dom = kernels[dom]["ms"] * 1e-3
    roofline = {"bound": "hbm", "kernel": dom,
                # headline: the bytes this layout has to move per launch (SELL
                # values, 2-byte row metadata, vectors; pattern rows carry no
                # column index), DESIGN.md §4
                "achieved": kernels[dom]["format_gbs"], "peak": peak, "unit": "GB/s",
                "frac": round(kernels[dom]["format_gbs"] / peak, 4),
                "bytes_per_launch": fb[dom], "bytes": "format bytes (DESIGN.md §4)",
                "traffic": traffic,
                "traffic_frac": round(traffic / t_dom / 1e9 / peak, 4) if traffic else None,
                "peak_source": peak_src,
                # SURVEY.md §8(d) CSR model: counts the column indices the
                # row-pattern layout never reads, so it can exceed 1
                "model_bytes_per_launch": kb[dom], "model_achieved": kernels[dom]["gbs"],
                "model_frac": kernels[dom]["frac"],
                "timing": "CUDA events around back-to-back launches chained by programmatic dependent "
                          "launch (as in the solve graph); kernels.*.ms_cold: one launch between two events"}
    it_med = int(np.median(iters))
    if wave:
        iter_bytes = kb["spmv_p"] + kb["wave"]
    else:
        iter_bytes = (max(cs.k - 2, 0) * kb["bjac_middle"] + (kb["bjac_last"] if cs.k > 1 else 0)
                      + (kb["spmv_p"] + kb["update_first"] if fused
                         else kb["pupdate"] + kb["spmv_pq"] + kb["bjac_first"] + kb["update"]))
    solve_gbs = world * iter_bytes * it_med / (ms_per_step * 1e-3) / 1e9

    # ---- CPU baseline (rank 0, N=1 only) -----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dt, its = cpu_sample(cs, part, policy, args.cpu_iters, 1)
        it_full = ref_iterations(cs.name, policy)
        src = "the reference-order iteration count of tests/golden/fullsize"
        if it_full is None:
            it_full, src = it_med, "the GPU's iteration count (no reference-order fixture)"
        cpu_solve = dt / its * it_full
        cpu = {"value": 1.0 / cpu_solve, "unit": "solve/s", "cores": 1, "kind": "port",
               "sample": f"{cs.name.upper()} solve capped at {its} iterations "
                         f"({dt:.1f} s; oracle restatement of the reference, reference dot "
                         f"order, 1 thread like the reference's numba kernels), "
                         f"scaled to the {it_full}-iteration solve ({src})",
               "host_cores": os.cpu_count()}
    if rank == 0:
        line = {
            "metric": metric_name(cs), "value": value, "unit": "solve/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64 CG / f32 preconditioner" if pp.needs_low else "f64",
            "data": "synthetic (seeded SplitMix64 fields per BASELINE.json configs)",
            "config": config_dict(cs, part, policy, {
                "parallelism": (f"z-slabs over {world} GPU(s), NCCL halos + fp64 all-reduce"
                                if sharded else "1 GPU"),
                "graph": ("one persistent cooperative kernel per solve (k_solve_small: at most one tile "
                          "per SM); kernels.* below time the three-kernel iteration it replaces"
                          if launches / max(args.steps, 1) < 16 and not sharded else
                          "one CUDA graph per solve: a device-side while loop over 16-iteration bodies"),
                "row_patterns": plan.layout_info()}),
            "iterations": it_med, "time_to_solution_ms": ms_per_step,
            "converged": bool(rep.converged), "final_true_relres": rep.final_true_relres,
            # north_star: final true fp64 relres at or below the tolerance
            # (C3 ends at 1.10e-9 > 1e-10, as the reference's own order does)
            "true_relres_met": bool(rep.final_true_relres <= cs.res_tol),
            "solve_gbs": round(solve_gbs, 1),
            "roofline": roofline, "kernels": kernels,
            "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    # NCCL's own log lines (e.g. "NCCL version ...") must not reach stdout,
    # where the driver reads exactly one JSON line
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_b200(args, world, rank, local)


if __name__ == "__main__":
    main()
