"""Preconditioned CG with per-iteration precision branching — on the GPU.

Drop-in for the reference's ``mpcg.solver`` (pkg/src/mpcg/solver.py:1-274).
``pcg_solve`` keeps the reference's signature, validation, exception
classes/messages, stopping rule (implicit relres <= res_tol) and report
fields, but the whole loop runs on the device (mpb_pcg_solve): the fused
preconditioner passes, the fused p-update+SpMV, the fused x/r update and
one-CTA scalar steps (rho, alpha, beta, relres, the aMP branch choice, error
flags, trace entries) are captured once as a CUDA graph of several
iterations and replayed until the device sets ``done``.  The host reads a
small pinned state block once per replay, never per kernel.

Arithmetic is the reference's, bit for bit, except the order of the three
fp64 dot products per iteration, which is the fixed tile-tree order of
include/mpbjac_order.h (reduction_mode "tree").
"""
from __future__ import annotations

import csv
import ctypes as C
import math
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib
from .device import dtype_name, is_tensor, to_device, to_host
from .policies import KIND_CODE, MixedPreconditioner, PrecisionPolicy
from .sparse import NarrowingOverflowError, PrecisionMismatchError, SparseMatrix, _narrow_error

#: smallest positive normal float64; zero residuals clamp here before log10
TINY = float(np.finfo(np.float64).tiny)


class SolverError(RuntimeError):
    """Base class for failures inside pcg_solve."""


class BreakdownError(SolverError):
    """r'z hit exactly zero with a nonzero residual."""


class IndefiniteOperatorError(SolverError):
    """A quadratic form that must stay positive went nonpositive."""


class NonFiniteResidualError(SolverError):
    """The residual norm left the finite range."""


@dataclass(frozen=True)
class SolveConfig:
    """Stopping rule and trace options for pcg_solve (solver.py:47-66)."""

    res_tol: float = 1e-10
    max_iter: int | None = None
    record_true_residual_every: int = 0

    def __post_init__(self):
        if not (self.res_tol > 0):
            raise ValueError("res_tol must be positive")
        if self.max_iter is not None and self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")
        if self.record_true_residual_every < 0:
            raise ValueError("record_true_residual_every must be >= 0")

    def iteration_cap(self, n: int) -> int:
        if self.max_iter is not None:
            return self.max_iter
        return min(10 * n, 20000)


@dataclass
class IterationRecord:
    """One PCG iteration: residual state and the branch that produced it."""

    iteration: int
    implicit_relres: float
    true_relres: float | None
    branch: str
    wall_time: float


@dataclass
class SolveReport:
    """Everything a solve produced, including the solution itself.

    ``stats`` (not in the reference) carries the device-side numbers:
    device loop seconds, kernel launches, r0 norm."""

    converged: bool
    iterations: int
    trace: list
    final_true_relres: float
    total_time: float
    policy: PrecisionPolicy
    x: object
    stats: dict = dc_field(default_factory=dict)


def _dev_struct(A: SparseMatrix, mp: MixedPreconditioner):
    """Device CSR shared by the SpMV and both preconditioner instances."""
    P = mp.any
    if A.values.dtype != np.float64:
        # the reference's spmv(A, p) with an fp32 A (sparse.py:50-54, 178)
        raise PrecisionMismatchError(
            f"spmv: operands mix precisions (float32, float64)")
    D = P.dcsr
    op = None  # the operator's SELL values when they are not the preconditioner's
    if P.source is not A:
        same = (P.source.n == A.n and np.array_equal(P.source.row_ptr, A.row_ptr)
                and np.array_equal(P.source.col_idx, A.col_idx))
        if not same:
            raise NotImplementedError(
                "GPU pcg_solve needs the preconditioner set up from a matrix "
                "with the solved matrix's sparsity structure")
        # The outer SpMV and the true residuals always multiply by the A
        # passed in (solver.py:154, 93-98); the preconditioner keeps the
        # values it was set up from.  Same structure: A's fp64 values are
        # packed into the preconditioner's SELL-32 layout once and cached.
        cache = A.__dict__.setdefault("_op_sell", {})
        hit = cache.get(id(D))
        if hit is None or hit[0] is not D:
            v = to_device(A.values, device=D.device)
            hit = (D, v, D.sell_values(v))
            cache[id(D)] = hit
        op = hit[2]
    val64 = mp.p_high.dvalues if mp.p_high is not None else None
    if val64 is None:
        if D.val64 is None:
            D.val64 = to_device(P.source.values.astype(np.float64), device=D.device)
        val64 = D.val64
    val32 = mp.p_low.dvalues if mp.p_low is not None else None
    s = D.c_struct(val64=val64, val32=val32, plan=P.plan)
    s.op_sell_val64 = op.data_ptr() if op is not None else None
    if op is not None:  # the operator's values in the plan's packed layout (offset-slot SpMV)
        s.op_ib_val64 = P.plan.inblock_values(op).data_ptr()
    return D, s


def true_relres(A: SparseMatrix, x, b, r0_norm: float) -> float:
    """||b - Ax|| / r0_norm, recomputed from scratch (solver.py:93-98),
    summed in device order."""
    if r0_norm == 0:
        raise ValueError("r0_norm must be nonzero")
    from .bjac import BlockPartition, DevicePlan
    h = _lib.Handle.get()
    D = A.device()
    if D.val64 is None:
        D.val64 = to_device(A.values.astype(np.float64), device=D.device)
    key = "_uniform_plan"
    plan = A.__dict__.get(key)
    if plan is None:
        plan = DevicePlan(h, BlockPartition.fixed_size(A.n, 512), A.row_ptr)
        A.__dict__[key] = plan
    xd, bd = to_device(x, "float64", D.device), to_device(b, "float64", D.device)
    s = D.c_struct()
    out = C.c_double()
    _lib.check(h.lib.mpb_true_relres(h.ptr, plan.ptr, C.byref(s), _lib.ptr(xd),
                                     _lib.ptr(bd), float(r0_norm), C.byref(out)),
               "true_relres")
    return float(out.value)


def _workspace(mp, plan, n, device, ghosts=0):
    torch = __import__("torch")
    ws = getattr(mp, "_workspace", None)
    if ws is None or ws[0] is not plan or ws[2] != ghosts:
        nbytes = int(_lib.load().mpb_solve_workspace_bytes_dist(plan.ptr, n, ghosts))
        if nbytes < 0:
            _lib.check(nbytes, "workspace")
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        ws = (plan, buf, ghosts)
        mp._workspace = ws
    return ws[1]


def _solve_buffers(mp, n, cap, device, ghosts=0):
    torch = __import__("torch")
    bufs = getattr(mp, "_solve_bufs", None)
    key = (n, cap, str(device), ghosts)
    if bufs is None or bufs[0] != key:
        f64 = dict(dtype=torch.float64, device=device)
        bufs = (key, torch.empty(n, **f64), torch.empty(n + ghosts, **f64),
                torch.empty((3, cap), **f64), torch.empty(cap, dtype=torch.int32, device=device))
        mp._solve_bufs = bufs
    return bufs[1:]


def pcg_solve(A: SparseMatrix, b, mp: MixedPreconditioner,
              config: SolveConfig = SolveConfig(), x0=None, *,
              graph_iters: int = 0) -> SolveReport:
    """Run PCG on Ax = b under the mixed preconditioner's policy
    (solver.py:101-184), entirely on the GPU.

    Raises BreakdownError / IndefiniteOperatorError / NonFiniteResidualError
    / NarrowingOverflowError when the iteration cannot continue; running out
    of iterations returns converged=False.  b (and x0) may be numpy arrays or
    CUDA tensors; x comes back in the same kind.
    """
    if A.n != A.m:
        raise ValueError(f"matrix is {A.n}x{A.m}, solver needs square")
    return _run_solve(A, b, mp, config, x0, graph_iters=graph_iters)


def _run_solve(A: SparseMatrix, b, mp: MixedPreconditioner, config: SolveConfig, x0=None,
               dist=None, n_global=None, graph_iters: int = 0, handle=None) -> SolveReport:
    """pcg_solve after the square check.  dist = (comm, halo, ghosts[,
    overflow hook]): this rank's slab of a multi-GPU solve
    (distributed.SlabSolver / LocalSlabGroup); handle: a private handle
    (in-process slab ranks), else the device's."""
    torch = __import__("torch")
    if tuple(b.shape) != (A.n,) or dtype_name(b) != "float64":
        raise ValueError(f"rhs must be float64 of shape ({A.n},)")
    if mp.n != A.n:
        raise ValueError(f"preconditioner is for {mp.n} rows, matrix has {A.n}")
    if x0 is not None and (tuple(x0.shape) != (A.n,) or dtype_name(x0) != "float64"):
        raise ValueError(f"x0 must be float64 of shape ({A.n},)")
    tensor_io = is_tensor(b)
    D, s = _dev_struct(A, mp)
    P = mp.any
    h = handle if handle is not None else _lib.Handle.get(D.device.index)
    cap = int(config.iteration_cap(A.n if n_global is None else n_global))
    ghosts = 0 if dist is None else int(dist[2])
    # persistent per-preconditioner buffers keep the device pointers stable,
    # so the captured CUDA graph is reused from one solve to the next
    bd, x_ext, tr, trb = _solve_buffers(mp, A.n, cap, D.device, ghosts)
    x = x_ext[:A.n]
    bd.copy_(b if is_tensor(b) else torch.from_numpy(np.ascontiguousarray(b)))
    if x0 is not None:
        x.copy_(x0 if is_tensor(x0) else torch.from_numpy(np.ascontiguousarray(x0)))
    ws = _workspace(mp, P.plan, A.n, D.device, ghosts)
    opt = _lib.MpbSolveOptions()
    opt.kind = KIND_CODE[mp.policy.kind]
    opt.adp_tol = float(mp.policy.adp_tol) if mp.policy.adp_tol is not None else 0.0
    opt.k, opt.t = P.k, P.t
    opt.res_tol = float(config.res_tol)
    opt.max_iter = cap
    opt.true_stride = int(config.record_true_residual_every)
    opt.has_x0 = 0 if x0 is None else 1
    opt.graph_iters = int(graph_iters)
    res = _lib.MpbSolveResult()
    if dist is None:
        _lib.check(h.lib.mpb_pcg_solve(
            h.ptr, P.plan.ptr, C.byref(s), C.byref(opt), _lib.ptr(bd), _lib.ptr(x_ext),
            _lib.ptr(tr[0]), _lib.ptr(tr[1]), _lib.ptr(trb), _lib.ptr(tr[2]),
            _lib.ptr(ws), ws.numel(), C.byref(res)), "pcg_solve")
    else:
        comm, halo = dist[0], dist[1]
        _lib.check(h.lib.mpb_pcg_solve_dist(
            h.ptr, comm, C.byref(halo), P.plan.ptr, C.byref(s), C.byref(opt), _lib.ptr(bd),
            _lib.ptr(x_ext), _lib.ptr(tr[0]), _lib.ptr(tr[1]), _lib.ptr(trb), _lib.ptr(tr[2]),
            _lib.ptr(ws), ws.numel(), C.byref(res)), "pcg_solve_dist")
    it = int(res.iterations)
    err = int(res.error)
    if err == _lib.SOLVE_NARROW_OVERFLOW and dist is not None and len(dist) > 3:
        dist[3](res)   # global first overflow index and value (multi-GPU)
    if err:
        _raise_solve_error(err, res)
    stats = {"device_seconds": float(res.device_seconds),
             "kernel_launches": int(res.kernel_launches),
             "r0_norm": float(res.r0_norm)}
    xo = x.clone() if tensor_io else to_host(x)
    if res.r0_norm == 0.0:
        return SolveReport(True, 0, [], 0.0, 0.0, mp.policy, xo, stats)
    trh = to_host(tr[:, :it])
    brh = to_host(trb[:it])
    trace = [IterationRecord(i + 1, float(trh[0, i]),
                             None if math.isnan(trh[1, i]) else float(trh[1, i]),
                             "high" if brh[i] == 0 else "low", float(trh[2, i]))
             for i in range(it)]
    return SolveReport(bool(res.converged), it, trace,
                       float(res.final_true_relres), float(res.device_seconds),
                       mp.policy, xo, stats)


def _raise_solve_error(err: int, res) -> None:
    it = int(res.err_iteration)
    v = float(res.err_value)
    if err == _lib.SOLVE_BREAKDOWN:
        raise BreakdownError(f"iteration {it}: r'z = 0 with nonzero residual")
    if err == _lib.SOLVE_INDEF_PRECOND:
        raise IndefiniteOperatorError(
            f"iteration {it}: r'z = {v!r} < 0, preconditioner is not positive "
            "definite here")
    if err == _lib.SOLVE_INDEF_MATRIX:
        raise IndefiniteOperatorError(
            f"iteration {it}: p'Ap = {v!r} <= 0, matrix is not positive "
            "definite on this direction")
    if err == _lib.SOLVE_NONFINITE:
        raise NonFiniteResidualError(f"iteration {it}: residual norm is {v!r}")
    if err == _lib.SOLVE_NARROW_OVERFLOW:
        raise _narrow_error("vector", int(res.overflow_count),
                            int(res.overflow_index), np.float64(v))
    raise SolverError(f"iteration {it}: solver error {err}")


# ---------------------------------------------------------------------------
# trace tooling (host side; solver.py:187-274)
# ---------------------------------------------------------------------------

def _relres_array(trace) -> np.ndarray:
    if len(trace) and isinstance(trace[0], IterationRecord):
        return np.array([rec.implicit_relres for rec in trace])
    return np.asarray(trace, dtype=np.float64)


def detect_divergence(trace_a, trace_b, delta_log10: float = 0.5) -> int | None:
    """1-based iteration where the two residual histories first differ by
    more than delta_log10 decades (common prefix only), else None."""
    a = _relres_array(trace_a)
    b = _relres_array(trace_b)
    m = min(a.size, b.size)
    if m == 0:
        return None
    gap = np.abs(np.log10(np.maximum(a[:m], TINY)) - np.log10(np.maximum(b[:m], TINY)))
    hit = np.flatnonzero(gap > delta_log10)
    return int(hit[0]) + 1 if hit.size else None


def speedup(report_uniform, report_mixed) -> float:
    """Wall-time ratio uniform/mixed; both runs must have converged."""
    if not (report_uniform.converged and report_mixed.converged):
        raise ValueError("speedup is only defined between converged runs")
    if report_mixed.total_time == 0:
        raise ValueError("mixed run reports zero time")
    return report_uniform.total_time / report_mixed.total_time


_CSV_HEADER = ["iteration", "implicit_relres", "true_relres", "branch", "wall_time"]


def trace_to_csv(report: SolveReport, path, include_timings: bool = False) -> None:
    """Iteration trace as CSV; wall_time is 0.0 unless include_timings, so
    identical reruns give identical files."""
    with open(path, "w", newline="", encoding="ascii") as fh:
        w = csv.writer(fh)
        w.writerow(_CSV_HEADER)
        for rec in report.trace:
            w.writerow([rec.iteration, repr(rec.implicit_relres),
                        "" if rec.true_relres is None else repr(rec.true_relres),
                        rec.branch,
                        repr(rec.wall_time) if include_timings else "0.0"])


def read_trace_csv(path) -> list:
    with open(path, "r", newline="", encoding="ascii") as fh:
        rows = csv.reader(fh)
        header = next(rows, None)
        if header != _CSV_HEADER:
            raise ValueError(f"{path}: not a trace file (header {header})")
        out = []
        for row in rows:
            if len(row) != 5:
                raise ValueError(f"{path}: malformed row {row!r}")
            out.append(IterationRecord(int(row[0]), float(row[1]),
                                       None if row[2] == "" else float(row[2]),
                                       row[3], float(row[4])))
    return out


def report_summary(report: SolveReport, extra: dict | None = None) -> dict:
    d = {"policy": report.policy.label(), "converged": report.converged,
         "iterations": report.iterations,
         "final_true_relres": report.final_true_relres,
         "total_time_s": report.total_time}
    if extra:
        d.update(extra)
    return d


def profile_iteration(A: SparseMatrix, mp: MixedPreconditioner, *,
                      config: SolveConfig = SolveConfig(), branch: str = "low",
                      reps: int = 20, ghosts: int = 0, n_global=None) -> dict:
    """Mean CUDA-event time (ms) per launch of each kernel of one PCG
    iteration, on the buffers pcg_solve uses (mpb_profile_iteration): each
    kernel launched alone ("<name>") and chained back to back with
    programmatic dependent launch as in the solve graph ("<name>_chained").
    Call after at least one pcg_solve with the same A / mp / config.
    ghosts > 0: a slab of a multi-GPU solve (local kernels only)."""
    D, s = _dev_struct(A, mp)
    P = mp.any
    h = _lib.Handle.get(D.device.index)
    cap = int(config.iteration_cap(A.n if n_global is None else n_global))
    bd, x, _, _ = _solve_buffers(mp, A.n, cap, D.device, ghosts)
    ws = _workspace(mp, P.plan, A.n, D.device, ghosts)
    opt = _lib.MpbSolveOptions()
    opt.kind = KIND_CODE[mp.policy.kind]
    opt.adp_tol = float(mp.policy.adp_tol) if mp.policy.adp_tol is not None else 0.0
    opt.k, opt.t = P.k, P.t
    opt.res_tol = float(config.res_tol)
    opt.max_iter = cap
    out = (C.c_double * 18)()
    if n_global is None:    # one GPU: the kernels pcg_solve runs (fused iteration)
        _lib.check(h.lib.mpb_profile_iteration(
            h.ptr, P.plan.ptr, C.byref(s), C.byref(opt), _lib.ptr(bd), _lib.ptr(x),
            _lib.ptr(ws), ws.numel(), 0 if branch == "high" else 1, int(reps), out),
            "profile_iteration")
    else:                   # a slab of a multi-GPU solve (unfused iteration)
        _lib.check(h.lib.mpb_profile_iteration_dist(
            h.ptr, P.plan.ptr, C.byref(s), C.byref(opt), int(ghosts), _lib.ptr(bd), _lib.ptr(x),
            _lib.ptr(ws), ws.numel(), 0 if branch == "high" else 1, int(reps), out),
            "profile_iteration")
    names = ("bjac_first", "bjac_middle", "bjac_last", "spmv_pq", "update",
             "update_first", "iteration", "pupdate")
    res = {k: float(out[i]) for i, k in enumerate(names)}
    res.update({k + "_chained": float(out[8 + i]) for i, k in enumerate(names)})
    res["wave"], res["wave_chained"] = float(out[16]), float(out[17])
    return res
