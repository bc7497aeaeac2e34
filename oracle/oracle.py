"""ctypes front end of the CPU oracle (oracle/mpbjac_oracle.c).

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline / ``--impl reference`` legs import this module,
and only as the checker or the CPU baseline.  The product package
(paper_2407_15973_b200) never imports it.

The kernel-level functions keep the reference's backend signatures
(pkg/src/mpcg/kernels_numba.py:18-70), so this module can itself be
monkeypatched into ``mpcg.backend.kernels`` to pin it against the reference
(tests/golden/make_golden.py does exactly that).  ``setup_arrays`` restates
bjac.setup (pkg/src/mpcg/bjac.py:152-190) and ``pcg_solve`` restates
solver.pcg_solve (pkg/src/mpcg/solver.py:101-184) with the policies of
pkg/src/mpcg/policies.py:102-183.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmpbjac_oracle.so")

reduction_mode = "sequential"

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_lib = None

KIND_CODE = {"uniform": 0, "fixed-low": 1, "adaptive-hl": 2, "adaptive-lh": 3}
ERR_NAMES = {0: None, 1: "breakdown", 2: "indefinite-preconditioner",
             3: "indefinite-matrix", 4: "nonfinite", 5: "narrowing-overflow",
             6: "bad-relres"}


class _Problem(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("rp", C.c_void_p), ("ci", C.c_void_p),
        ("val64", C.c_void_p), ("val32", C.c_void_p),
        ("diag64", C.c_void_p), ("diag32", C.c_void_p),
        ("in_block", C.c_void_p), ("k", C.c_int), ("t", C.c_int),
        ("kind", C.c_int), ("adp_tol", C.c_double), ("res_tol", C.c_double),
        ("cap", C.c_int64), ("stride", C.c_int64), ("order", C.c_int),
        ("ntiles", C.c_int64), ("tile_lo", C.c_void_p),
        ("pval64", C.c_void_p),
    ]


class _Result(C.Structure):
    _fields_ = [
        ("converged", C.c_int), ("iterations", C.c_int64),
        ("final_true_relres", C.c_double), ("r0_norm", C.c_double),
        ("error", C.c_int), ("err_it", C.c_int64), ("err_val", C.c_double),
        ("overflow_count", C.c_int64), ("overflow_index", C.c_int64),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc only; no GPU needed)."""
    srcs = [os.path.join(_HERE, "mpbjac_oracle.c"),
            os.path.join(os.path.dirname(_HERE), "include", "mpbjac_order.h")]
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(f) for f in srcs):
        subprocess.run(["make", "-s", "-C", _HERE, "libmpbjac_oracle.so"],
                       check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        for suf, fp in (("f64", _f64p), ("f32", _f32p)):
            getattr(L, f"orc_csr_matvec_{suf}").argtypes = [
                C.c_int64, _i64p, _i32p, fp, fp, fp]
            getattr(L, f"orc_sweeps_{suf}").argtypes = [
                _i64p, _i32p, fp, _u8p, fp, C.c_int, fp, fp, fp,
                C.c_int64, C.c_int64]
            getattr(L, f"orc_dot_seq_{suf}").argtypes = [C.c_int64, fp, fp]
            getattr(L, f"orc_dot_seq_{suf}").restype = (
                C.c_double if suf == "f64" else C.c_float)
            getattr(L, f"orc_norm_sq_{suf}").argtypes = [C.c_int64, fp]
            getattr(L, f"orc_norm_sq_{suf}").restype = C.c_double
            getattr(L, f"orc_bjac_apply_{suf}").argtypes = [
                C.c_int64, _i64p, _i32p, fp, _u8p, fp, C.c_int, C.c_int,
                fp, fp, fp]
        L.orc_narrow.argtypes = [C.c_int64, _f64p, _f32p,
                                 C.POINTER(C.c_int64)]
        L.orc_narrow.restype = C.c_int64
        L.orc_plan_tiles.argtypes = [C.c_int64, _i64p, _i64p, _i64p,
                                     C.POINTER(C.c_int)]
        L.orc_plan_tiles.restype = C.c_int64
        L.orc_tree_sum.argtypes = [C.c_int64, _i64p, _f64p]
        L.orc_tree_sum.restype = C.c_double
        L.orc_tree_dot.argtypes = [C.c_int64, C.c_int64, _i64p, _f64p, _f64p]
        L.orc_tree_dot.restype = C.c_double
        L.orc_pcg_solve.argtypes = [C.POINTER(_Problem), _f64p, C.c_int,
                                    _f64p, _f64p, _f64p,
                                    np.ctypeslib.ndpointer(np.int32),
                                    C.POINTER(_Result)]
        L.orc_pcg_solve.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_get_threads.restype = C.c_int
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def _suf(arr):
    if arr.dtype == np.float64:
        return "f64"
    if arr.dtype == np.float32:
        return "f32"
    raise TypeError(f"unsupported dtype {arr.dtype}")


# --- the reference's backend kernel signatures (kernels_numba.py) ----------

def csr_matvec(row_ptr, col_idx, values, x, out):
    getattr(lib(), f"orc_csr_matvec_{_suf(values)}")(
        out.size, np.ascontiguousarray(row_ptr, np.int64),
        np.ascontiguousarray(col_idx, np.int32), values, x, out)


def block_jacobi_sweeps(row_ptr, col_idx, values, in_block, diag, t,
                        r, y, tmp, row_start, row_end):
    getattr(lib(), f"orc_sweeps_{_suf(values)}")(
        np.ascontiguousarray(row_ptr, np.int64),
        np.ascontiguousarray(col_idx, np.int32), values,
        np.ascontiguousarray(in_block).view(np.uint8), diag, int(t),
        np.ascontiguousarray(r), y, tmp, int(row_start), int(row_end))


def dot_seq(x, y):
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    v = getattr(lib(), f"orc_dot_seq_{_suf(x)}")(x.size, x, y)
    return x.dtype.type(v)


def norm_sq_f64(x):
    x = np.ascontiguousarray(x)
    return float(getattr(lib(), f"orc_norm_sq_{_suf(x)}")(x.size, x))


# --- setup / apply / solve ---------------------------------------------------

def narrow(r):
    """(r32, count, first_bad) — sparse.py:202-214."""
    r = np.ascontiguousarray(r, np.float64)
    out = np.empty(r.size, np.float32)
    fb = C.c_int64(-1)
    cnt = lib().orc_narrow(r.size, r, out, C.byref(fb))
    return out, int(cnt), int(fb.value)


def setup_arrays(row_ptr, col_idx, values64, offsets):
    """diag64, diag32, val32, in_block as bjac.setup computes them
    (pkg/src/mpcg/bjac.py:171-188).  Raises ValueError like the reference."""
    row_ptr = np.asarray(row_ptr, np.int64)
    col_idx = np.asarray(col_idx, np.int32)
    n = row_ptr.size - 1
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    diag_pos = np.flatnonzero(rows == col_idx)
    if diag_pos.size != n:
        have = np.zeros(n, bool)
        have[rows[diag_pos]] = True
        raise ValueError(
            f"row {int(np.flatnonzero(~have)[0])} has no stored diagonal entry")
    with np.errstate(over="ignore"):
        val32 = values64.astype(np.float32)
    diag64 = values64[diag_pos].copy()
    diag32 = val32[diag_pos].copy()
    offsets = np.asarray(offsets, np.int64)
    blk = np.searchsorted(offsets, np.arange(n), side="right") - 1
    in_block = (blk[rows] == blk[col_idx]).astype(np.uint8)
    return diag64, diag32, val32, in_block


def bjac_apply(row_ptr, col_idx, values, in_block, diag, k, t, r):
    """BjacPreconditioner.apply (bjac.py:127-149) in values' precision."""
    values = np.ascontiguousarray(values)
    r = np.ascontiguousarray(r, values.dtype)
    n = r.size
    z = np.empty(n, values.dtype)
    work = np.empty(3 * n, values.dtype)
    getattr(lib(), f"orc_bjac_apply_{_suf(values)}")(
        n, np.ascontiguousarray(row_ptr, np.int64),
        np.ascontiguousarray(col_idx, np.int32), values,
        np.ascontiguousarray(in_block, np.uint8),
        np.ascontiguousarray(diag, values.dtype), int(k), int(t), r, z, work)
    return z


def plan_tiles(offsets, row_ptr):
    """(tile_lo int64[ntiles+1], large) per include/mpbjac_order.h."""
    offsets = np.ascontiguousarray(offsets, np.int64)
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    nb = offsets.size - 1
    n = int(offsets[-1])
    out = np.empty(nb + n // 256 + 2, np.int64)
    large = C.c_int(0)
    nt = lib().orc_plan_tiles(nb, offsets, row_ptr, out, C.byref(large))
    return out[:nt + 1].copy(), bool(large.value)


def tree_sum(tile_lo, vals):
    tile_lo = np.ascontiguousarray(tile_lo, np.int64)
    return float(lib().orc_tree_sum(tile_lo.size - 1, tile_lo,
                                    np.ascontiguousarray(vals, np.float64)))


def tree_dot(tile_lo, x, y):
    tile_lo = np.ascontiguousarray(tile_lo, np.int64)
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return float(lib().orc_tree_dot(x.size, tile_lo.size - 1, tile_lo, x, y))


def pcg_solve(row_ptr, col_idx, values, b, offsets, kind="uniform",
              adp_tol=None, k=2, t=2, res_tol=1e-10, max_iter=None,
              stride=0, order="sequential", x0=None, threads=None,
              prec_values=None):
    """Oracle solve.  order='sequential' replays the reference (numba) dot
    order, order='device' the GPU tile-tree order.  Returns a dict.
    prec_values: the preconditioner's source values (same structure), when
    it was set up from another matrix than the solved one."""
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col_idx = np.ascontiguousarray(col_idx, np.int32)
    values = np.ascontiguousarray(values, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    n = b.size
    offsets = np.ascontiguousarray(offsets, np.int64)
    pvals = values if prec_values is None else np.ascontiguousarray(prec_values, np.float64)
    diag64, diag32, val32, in_block = setup_arrays(row_ptr, col_idx, pvals,
                                                   offsets)
    tile_lo, _ = plan_tiles(offsets, row_ptr)
    cap = int(max_iter) if max_iter is not None else min(10 * n, 20000)
    if adp_tol is None:
        adp_tol = {"adaptive-hl": 10.0, "adaptive-lh": 1e-5}.get(kind, 0.0)
    P = _Problem()
    keep = (row_ptr, col_idx, values, val32, diag64, diag32, in_block, tile_lo, pvals)
    P.n = n
    P.rp, P.ci, P.val64, P.val32 = (a.ctypes.data for a in keep[:4])
    P.diag64, P.diag32, P.in_block = (a.ctypes.data for a in keep[4:7])
    P.k, P.t = int(k), int(t)
    P.kind = KIND_CODE[kind]
    P.adp_tol = float(adp_tol)
    P.res_tol = float(res_tol)
    P.cap = cap
    P.stride = int(stride)
    P.order = 0 if order == "sequential" else 1
    P.ntiles = tile_lo.size - 1
    P.tile_lo = tile_lo.ctypes.data
    P.pval64 = None if prec_values is None else pvals.ctypes.data
    x = np.zeros(n) if x0 is None else np.array(x0, np.float64)
    rel = np.zeros(cap)
    tru = np.full(cap, np.nan)
    br = np.zeros(cap, np.int32)
    R = _Result()
    if threads is not None:
        set_threads(threads)
    lib().orc_pcg_solve(C.byref(P), b, 0 if x0 is None else 1, x, rel, tru,
                        br, C.byref(R))
    del keep
    it = int(R.iterations)
    return {
        "x": x, "iterations": it, "converged": bool(R.converged),
        "relres": rel[:it].copy(), "true_relres": tru[:it].copy(),
        "branch": ["high" if v == 0 else "low" for v in br[:it]],
        "final_true_relres": float(R.final_true_relres),
        "r0_norm": float(R.r0_norm), "error": ERR_NAMES[int(R.error)],
        "err_it": int(R.err_it), "err_val": float(R.err_val),
        "overflow_count": int(R.overflow_count),
        "overflow_index": int(R.overflow_index),
    }
