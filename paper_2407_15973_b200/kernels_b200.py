"""The reference's kernel-backend plugin API, served by libmpbjac.so.

Signature-compatible with the reference's ``mpcg.kernels_numba`` /
``mpcg.kernels_numpy`` (pkg/src/mpcg/kernels_numba.py:15-115): host numpy
arrays in, results written in place.  Each call copies its operands to the
GPU and back, so this module is a parity harness (it lets the reference's
own tests run against the B200 kernels by monkeypatching
``mpcg.backend.kernels``, as pkg/tests/conftest.py:8-17 does), not the
solve path — ``solver.pcg_solve`` keeps everything resident.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .device import to_device, to_host

#: dots are summed in the fixed device tile-tree order (include/mpbjac_order.h)
reduction_mode = "tree"


def _h():
    return _lib.Handle.get()


def _suffix(values):
    if values.dtype == np.float64:
        return "f64"
    if values.dtype == np.float32:
        return "f32"
    raise TypeError(f"unsupported dtype {values.dtype}")


def csr_matvec(row_ptr, col_idx, values, x, out):
    """out = A @ x, row-sequential accumulation (kernels_numba.py:37-45)."""
    h = _h()
    n = out.size
    rp = to_device(np.asarray(row_ptr).astype(np.int32))
    ci = to_device(np.asarray(col_idx, np.int32))
    v = to_device(np.asarray(values))
    xd = to_device(np.asarray(x, values.dtype))
    yd = to_device(np.empty(n, values.dtype))
    fn = getattr(h.lib, f"mpb_csr_matvec_{_suffix(values)}")
    _lib.check(fn(h.ptr, n, _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(v), _lib.ptr(xd),
                  _lib.ptr(yd)), "csr_matvec")
    out[:] = to_host(yd)


def block_jacobi_sweeps(row_ptr, col_idx, values, in_block, diag, t, r, y, tmp,
                        row_start, row_end):
    """t masked Jacobi sweeps on rows [row_start, row_end)
    (kernels_numba.py:48-70); y and tmp are updated in place."""
    h = _h()
    rp = to_device(np.asarray(row_ptr).astype(np.int32))
    ci = to_device(np.asarray(col_idx, np.int32))
    v = to_device(np.asarray(values))
    mask = to_device(np.asarray(in_block).astype(np.uint8))
    dg = to_device(np.asarray(diag, values.dtype))
    rd = to_device(np.asarray(r, values.dtype))
    yd = to_device(np.asarray(y))
    td = to_device(np.asarray(tmp))
    fn = getattr(h.lib, f"mpb_block_jacobi_sweeps_{_suffix(values)}")
    _lib.check(fn(h.ptr, _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(v), _lib.ptr(mask),
                  _lib.ptr(dg), int(t), _lib.ptr(rd), _lib.ptr(yd), _lib.ptr(td),
                  int(row_start), int(row_end)), "block_jacobi_sweeps")
    y[:] = to_host(yd)
    tmp[:] = to_host(td)


def dot_seq(x, y):
    """Dot product in the operand dtype (device tile-tree order)."""
    h = _h()
    x = np.ascontiguousarray(x)
    xd, yd = to_device(x), to_device(np.asarray(y, x.dtype))
    if x.dtype == np.float64:
        out = C.c_double()
        _lib.check(h.lib.mpb_dot_f64(h.ptr, None, x.size, _lib.ptr(xd), _lib.ptr(yd),
                                     C.byref(out)), "dot")
        return np.float64(out.value)
    out32 = C.c_float()
    _lib.check(h.lib.mpb_dot_f32(h.ptr, None, x.size, _lib.ptr(xd), _lib.ptr(yd),
                                 C.byref(out32)), "dot")
    return np.float32(out32.value)


def norm_sq_f64(x):
    """Sum of squares with each element widened to float64."""
    h = _h()
    x = np.ascontiguousarray(x)
    xd = to_device(x)
    out = C.c_double()
    fn = h.lib.mpb_norm_sq_f64 if x.dtype == np.float64 else h.lib.mpb_norm_sq_f32
    _lib.check(fn(h.ptr, None, x.size, _lib.ptr(xd), C.byref(out)), "norm_sq_f64")
    return float(out.value)


def fill_stencil(n, fxm, fxp, fym, fyp, fzm, fzp, inv_h2, row_ptr, col_idx, values):
    """7-point CSR fill from face arrays (kernels_numba.py:73-115).  Setup-time
    assembly, host side (see problems.stencil_csr)."""
    from .problems import stencil_csr
    rp, ci, v = stencil_csr(int(n), (fxm, fxp, fym, fyp, fzm, fzp), float(inv_h2))
    if not np.array_equal(rp, np.asarray(row_ptr)):
        raise ValueError("row_ptr does not match the 7-point structure")
    col_idx[:] = ci
    values[:] = v
