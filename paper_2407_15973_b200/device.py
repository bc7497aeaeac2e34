"""Device-resident CSR and host<->device helpers.

Layout in HBM: int32 ``row_ptr`` (n+1) and
``col_idx`` (nnz), fp64 values (A and the fp64 preconditioner instance share
one buffer, because setup's fp64 "conversion" is a bitwise copy,
pkg/src/mpcg/bjac.py:175 + sparse.py:203-204), and an fp32 values copy for
the low-precision instance.  PyTorch only allocates; every computation goes
through libmpbjac.so.
"""
from __future__ import annotations

import numpy as np

from . import _lib


def torch():
    import torch as _t
    return _t


def default_device():
    t = torch()
    if not t.cuda.is_available():
        raise _lib.BackendUnavailableError(
            "no CUDA device visible: the B200 kernels have no CPU fallback")
    return t.device("cuda", t.cuda.current_device())


def is_tensor(x) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, _t.Tensor)


_NP2T = {np.dtype(np.float64): "float64", np.dtype(np.float32): "float32",
         np.dtype(np.int32): "int32", np.dtype(np.int64): "int64",
         np.dtype(np.uint8): "uint8", np.dtype(np.bool_): "bool"}


def to_device(x, dtype=None, device=None):
    """Contiguous CUDA tensor holding x (numpy array or tensor)."""
    t = torch()
    dev = device if device is not None else default_device()
    if is_tensor(x):
        y = x.to(device=dev)
        if dtype is not None:
            y = y.to(getattr(t, dtype))
        return y.contiguous()
    a = np.ascontiguousarray(x if dtype is None else np.asarray(x, dtype=dtype))
    return t.from_numpy(a).to(dev, non_blocking=False)


def to_host(t):
    return t.detach().cpu().numpy()


def dtype_name(x) -> str:
    if is_tensor(x):
        return str(x.dtype).replace("torch.", "")
    return str(np.asarray(x).dtype)


class DeviceSell:
    """SELL-32 structure of a DeviceCSR (library-owned mpb_sell)."""

    def __init__(self, handle, n, host_row_ptr, row_ptr, col_idx):
        import ctypes as C
        self.h = handle
        self.ptr = C.c_void_p()
        hrp = np.ascontiguousarray(host_row_ptr, np.int64)
        _lib.check(handle.lib.mpb_sell_create(
            handle.ptr, int(n), hrp.ctypes.data_as(C.c_void_p),
            _lib.ptr(row_ptr), _lib.ptr(col_idx), C.byref(self.ptr)), "mpb_sell_create")
        self.nnz = int(handle.lib.mpb_sell_nnz(self.ptr))

    def __del__(self):
        try:
            if self.ptr:
                self.h.lib.mpb_sell_destroy(self.ptr)
        except Exception:  # interpreter shutdown
            pass


class DeviceCSR:
    """CSR matrix resident on one GPU (int32 indices), plus its SELL-32
    layout (the hot kernels' format), built on first use."""

    def __init__(self, n, m, row_ptr, col_idx, val64=None, val32=None, host_row_ptr=None):
        self.n = int(n)
        self.m = int(m)
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.val64 = val64
        self.val32 = val32
        self.nnz = int(col_idx.numel())
        self.device = row_ptr.device
        self.host_row_ptr = host_row_ptr
        self.sell = None
        self._sell_vals = {}

    @classmethod
    def from_host(cls, n, m, row_ptr, col_idx, values, device=None):
        row_ptr = np.asarray(row_ptr)
        nnz = int(row_ptr[-1]) if row_ptr.size else 0
        if n >= 2 ** 31 - 1 or nnz >= 2 ** 31:
            raise ValueError("matrix too large for the int32-indexed device CSR")
        rp = to_device(row_ptr.astype(np.int32, copy=False), device=device)
        ci = to_device(np.asarray(col_idx, np.int32), device=device)
        values = np.asarray(values)
        hrp = np.asarray(row_ptr, np.int64)
        if values.dtype == np.float64:
            return cls(n, m, rp, ci, val64=to_device(values, device=device), host_row_ptr=hrp)
        return cls(n, m, rp, ci, val32=to_device(values, device=device), host_row_ptr=hrp)

    def _ensure_sell(self, handle):
        if self.sell is None:
            hrp = self.host_row_ptr
            if hrp is None:
                hrp = self.row_ptr.cpu().numpy().astype(np.int64)
            self.sell = DeviceSell(handle, self.n, hrp, self.row_ptr, self.col_idx)
        return self.sell

    def sell_values(self, values):
        """SELL-32 packing of a CSR value tensor of this matrix (cached)."""
        if values is None:
            return None
        key = (values.data_ptr(), str(values.dtype))
        packed = self._sell_vals.get(key)
        if packed is None:
            t = torch()
            h = _lib.Handle.get(self.device.index)
            S = self._ensure_sell(h)
            packed = t.empty(max(S.nnz, 1), dtype=values.dtype, device=self.device)
            fn = h.lib.mpb_sell_pack_f64 if values.dtype == t.float64 else h.lib.mpb_sell_pack_f32
            _lib.check(fn(h.ptr, S.ptr, _lib.ptr(self.row_ptr), _lib.ptr(values), _lib.ptr(packed)),
                       "mpb_sell_pack")
            self._sell_vals[key] = (values, packed)
        else:
            packed = packed[1]
        return packed

    def c_struct(self, val64=None, val32=None, plan=None) -> _lib.MpbCsr:
        s = _lib.MpbCsr()
        s.n = self.n
        s.nnz = self.nnz
        s.row_ptr = self.row_ptr.data_ptr()
        s.col_idx = self.col_idx.data_ptr()
        v64 = val64 if val64 is not None else self.val64
        v32 = val32 if val32 is not None else self.val32
        s.val64 = v64.data_ptr() if v64 is not None else None
        s.val32 = v32.data_ptr() if v32 is not None else None
        h = _lib.Handle.get(self.device.index)
        S = self._ensure_sell(h)
        s.sell = S.ptr
        sv64 = self.sell_values(v64)
        sv32 = self.sell_values(v32)
        s.sell_val64 = sv64.data_ptr() if sv64 is not None else None
        s.sell_val32 = sv32.data_ptr() if sv32 is not None else None
        if plan is not None:
            iv64 = plan.inblock_values(sv64)
            iv32 = plan.inblock_values(sv32)
            s.ib_val64 = iv64.data_ptr() if iv64 is not None else None
            s.ib_val32 = iv32.data_ptr() if iv32 is not None else None
        return s

    def nbytes(self) -> int:
        b = self.row_ptr.numel() * 4 + self.col_idx.numel() * 4
        for v in (self.val64, self.val32):
            if v is not None:
                b += v.numel() * v.element_size()
        if self.sell is not None:
            b += self.sell.nnz * 4
        for _, packed in self._sell_vals.values():
            b += packed.numel() * packed.element_size()
        return b
