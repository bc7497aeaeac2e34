"""Block-Jacobi preconditioner of k outer passes x t inner Jacobi sweeps.

Drop-in for the reference's ``mpcg.bjac`` (pkg/src/mpcg/bjac.py:1-190): same
``BlockPartition``, ``BjacPreconditioner`` (``apply``, ``inner_apply``) and
``setup`` signatures, checks and messages.  The difference is where the work
happens: setup converts and checks values on the GPU (mpb_convert_values_f32,
mpb_setup_diag_*), builds the device tile plan (mpb_plan_create), and
``apply`` is k launches of the fused tile kernel (mpb_bjac_apply_*): each
CTA stages whole blocks' CSR rows in shared memory with TMA bulk copies and
runs all t inner sweeps there.  The in-block mask of the reference
(bjac.py:187-188) is never materialised; it is derived from the block
bounds.  Results are bit-identical to the reference's numba kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import dtype_name, is_tensor, to_device, to_host
from .sparse import (NarrowingOverflowError, Precision, PrecisionMismatchError,
                     SparseMatrix, _narrow_error)


@dataclass(frozen=True)
class BlockPartition:
    """Contiguous row blocks given by ascending offsets (first 0, last n)."""

    offsets: np.ndarray

    def __post_init__(self):
        offs = np.ascontiguousarray(self.offsets, dtype=np.int64)
        object.__setattr__(self, "offsets", offs)
        if offs.ndim != 1 or offs.size < 2:
            raise ValueError("partition needs at least one block")
        if offs[0] != 0:
            raise ValueError("partition must start at row 0")
        if np.any(offs[1:] <= offs[:-1]):
            raise ValueError("partition offsets must be strictly increasing")

    @classmethod
    def equal_split(cls, n: int, nb: int) -> "BlockPartition":
        """nb contiguous blocks whose sizes differ by at most one."""
        if nb < 1:
            raise ValueError("need at least one block")
        if nb > n:
            raise ValueError(f"cannot split {n} rows into {nb} blocks")
        q, rem = divmod(n, nb)
        sizes = np.full(nb, q, dtype=np.int64)
        sizes[:rem] += 1
        return cls(np.concatenate(([0], np.cumsum(sizes))))

    @classmethod
    def fixed_size(cls, n: int, size: int) -> "BlockPartition":
        """Blocks of `size` rows (the last one may be shorter); the 64-row /
        96-row partitions of the benchmark configs."""
        if size < 1:
            raise ValueError("block size must be positive")
        offs = np.arange(0, n, size, dtype=np.int64)
        return cls(np.append(offs, n))

    @property
    def num_blocks(self) -> int:
        return self.offsets.size - 1

    @property
    def n(self) -> int:
        return int(self.offsets[-1])

    def block_range(self, b: int) -> tuple[int, int]:
        if not 0 <= b < self.num_blocks:
            raise IndexError(f"block {b} out of range")
        return int(self.offsets[b]), int(self.offsets[b + 1])

    def block_of_rows(self) -> np.ndarray:
        """Block id of every row, length n."""
        return np.searchsorted(self.offsets, np.arange(self.n), side="right") - 1


class DevicePlan:
    """Owns an mpb_plan (tile plan + block tables on the device)."""

    def __init__(self, handle, partition: BlockPartition, row_ptr: np.ndarray):
        self.h = handle
        self.ptr = C.c_void_p()
        offs = np.ascontiguousarray(partition.offsets, np.int64)
        rp = np.ascontiguousarray(row_ptr, np.int64)
        _lib.check(handle.lib.mpb_plan_create(
            handle.ptr, partition.n, partition.num_blocks,
            offs.ctypes.data_as(C.c_void_p), rp.ctypes.data_as(C.c_void_p),
            C.byref(self.ptr)), "mpb_plan_create")
        self.bound = None
        nt, large, mx = C.c_int64(), C.c_int(), C.c_int64()
        handle.lib.mpb_plan_info(self.ptr, C.byref(nt), C.byref(large), C.byref(mx))
        self.ntiles = int(nt.value)
        self.large = bool(large.value)
        self.max_tile_nnz = int(mx.value)

    def inblock_values(self, sell_values):
        """In-block SELL packing of SELL-32 values (cached per tensor)."""
        if sell_values is None:
            return None
        torch = __import__("torch")
        cache = self.__dict__.setdefault("_ib", {})
        key = (sell_values.data_ptr(), str(sell_values.dtype))
        hit = cache.get(key)
        if hit is None:
            nnz = int(self.h.lib.mpb_plan_inblock_nnz(self.ptr))
            if nnz < 0:
                _lib.check(nnz, "mpb_plan_inblock_nnz")
            out = torch.empty(max(nnz, 1), dtype=sell_values.dtype, device=sell_values.device)
            fn = (self.h.lib.mpb_plan_pack_inblock_f64 if sell_values.dtype == torch.float64
                  else self.h.lib.mpb_plan_pack_inblock_f32)
            _lib.check(fn(self.h.ptr, self.ptr, _lib.ptr(sell_values), _lib.ptr(out)),
                       "mpb_plan_pack_inblock")
            hit = (sell_values, out)
            cache[key] = hit
        return hit[1]

    def bind(self, dcsr) -> "DevicePlan":
        """Build the per-row static structure against the matrix's SELL-32
        layout (mpb_plan_bind_sell)."""
        S = dcsr._ensure_sell(self.h)
        if self.bound is not S:
            _lib.check(self.h.lib.mpb_plan_bind_sell(self.h.ptr, self.ptr, S.ptr), "mpb_plan_bind_sell")
            self.bound = S
        return self

    def layout_info(self) -> dict:
        """Row patterns of the bound structure ({"patterns", "generic_rows"}) and its
        offset-slot layout ("offset_slots": 7 or 0, "inblock_slots" mask,
        "offset_slot_update": the fused update runs on it too)."""
        npat, ngen = C.c_int(), C.c_int64()
        _lib.check(self.h.lib.mpb_plan_layout_info(self.ptr, C.byref(npat), C.byref(ngen)),
                   "mpb_plan_layout_info")
        slots, inb, near = C.c_int(), C.c_int(), C.c_int()
        _lib.check(self.h.lib.mpb_plan_offset_slot_info(self.ptr, C.byref(slots), C.byref(inb), C.byref(near)),
                   "mpb_plan_offset_slot_info")
        return {"patterns": int(npat.value), "generic_rows": int(ngen.value),
                "offset_slots": int(slots.value), "inblock_slots": int(inb.value),
                "offset_slot_update": bool(near.value)}

    def __del__(self):
        try:
            if self.ptr:
                self.h.lib.mpb_plan_destroy(self.ptr)
                self.ptr = C.c_void_p()
        except Exception:  # interpreter shutdown
            pass


@dataclass(eq=False)
class BjacPreconditioner:
    """Frozen result of setup(); apply and inner_apply do the work.

    Device state: ``dcsr`` (structure shared with the source matrix),
    ``dvalues`` (storage precision; for F64 the source matrix's own buffer),
    ``ddiag`` and ``plan``.  The reference's host attributes (row_ptr,
    col_idx, values, diag, in_block) are available as read-only properties.
    """

    partition: BlockPartition
    k: int
    t: int
    precision: Precision
    source: SparseMatrix
    dcsr: object
    dvalues: object
    ddiag: object
    plan: DevicePlan

    @property
    def n(self) -> int:
        return self.partition.n

    # reference-compatible host views ------------------------------------
    @property
    def row_ptr(self) -> np.ndarray:
        return self.source.row_ptr

    @property
    def col_idx(self) -> np.ndarray:
        return self.source.col_idx

    @property
    def values(self) -> np.ndarray:
        return to_host(self.dvalues)

    @property
    def diag(self) -> np.ndarray:
        return to_host(self.ddiag)

    @property
    def in_block(self) -> np.ndarray:
        blk = self.partition.block_of_rows()
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        return blk[rows] == blk[self.col_idx]

    def _csr_struct(self):
        if self.precision is Precision.F64:
            return self.dcsr.c_struct(val64=self.dvalues, val32=None, plan=self.plan)
        return self.dcsr.c_struct(val64=None, val32=self.dvalues, plan=self.plan)

    def _check_vector(self, r):
        if tuple(r.shape) != (self.n,):
            raise ValueError(f"vector has shape {tuple(r.shape)}, expected ({self.n},)")
        if dtype_name(r) != str(self.precision.dtype):
            raise PrecisionMismatchError(
                f"apply: vector is {dtype_name(r)}, preconditioner stores "
                f"{self.precision.dtype}")
        return r

    def apply(self, r):
        """z approximating (block diag A)^{-1} r, all in storage precision
        (bjac.py:127-149).  One fused kernel launch per outer pass."""
        torch = __import__("torch")
        r = self._check_vector(r if is_tensor(r) else np.asarray(r))
        h = _lib.Handle.get(self.dcsr.device.index)
        rd = to_device(r, device=self.dcsr.device)
        z = torch.empty_like(rd)
        s = self._csr_struct()
        fn = h.lib.mpb_bjac_apply_f64 if self.precision is Precision.F64 else h.lib.mpb_bjac_apply_f32
        _lib.check(fn(h.ptr, self.plan.ptr, C.byref(s), self.k, self.t,
                      _lib.ptr(rd), _lib.ptr(z)), "apply")
        return z if is_tensor(r) else to_host(z)

    def inner_apply(self, b: int, r_b):
        """t Jacobi sweeps on block b alone (bjac.py:106-125)."""
        torch = __import__("torch")
        start, end = self.partition.block_range(b)
        r_b = r_b if is_tensor(r_b) else np.asarray(r_b)
        if tuple(r_b.shape) != (end - start,):
            raise ValueError(f"block {b} has {end - start} rows, "
                             f"got vector of shape {tuple(r_b.shape)}")
        if dtype_name(r_b) != str(self.precision.dtype):
            raise PrecisionMismatchError(
                f"inner_apply: vector is {dtype_name(r_b)}, preconditioner stores "
                f"{self.precision.dtype}")
        h = _lib.Handle.get(self.dcsr.device.index)
        rd = to_device(r_b, device=self.dcsr.device)
        y = torch.empty_like(rd)
        s = self._csr_struct()
        fn = (h.lib.mpb_bjac_inner_apply_f64 if self.precision is Precision.F64
              else h.lib.mpb_bjac_inner_apply_f32)
        _lib.check(fn(h.ptr, C.byref(s), start, end, self.t, _lib.ptr(rd),
                      _lib.ptr(y)), "inner_apply")
        return y if is_tensor(r_b) else to_host(y)


def _device_values(A: SparseMatrix, precision: Precision, h):
    """Storage-precision values on the GPU, with the reference's narrowing
    overflow error (bjac.py:175 -> sparse.py:202-214)."""
    torch = __import__("torch")
    D = A.device()
    if A.values.dtype == np.float64:
        if precision is Precision.F64:
            return D, D.val64          # bitwise copy == shared buffer
        if D.val32 is None:
            out = torch.empty(D.nnz + 4, dtype=torch.float32, device=D.device)[:D.nnz]
            cnt, first = C.c_int64(), C.c_int64()
            _lib.check(h.lib.mpb_convert_values_f32(
                h.ptr, D.nnz, _lib.ptr(D.val64), _lib.ptr(out), C.byref(cnt),
                C.byref(first)), "setup")
            if cnt.value:
                k = int(first.value)
                raise _narrow_error("vector", int(cnt.value), k, np.float64(A.values[k]))
            D.val32 = out
        return D, D.val32
    # fp32 source matrix
    if precision is Precision.F32:
        return D, D.val32
    if D.val64 is None:
        out = torch.empty(D.nnz, dtype=torch.float64, device=D.device)
        _lib.check(h.lib.mpb_widen_f32_f64(h.ptr, D.nnz, _lib.ptr(D.val32), _lib.ptr(out)), "setup")
        D.val64 = out
    return D, D.val64


def _shared_plan(h, A: SparseMatrix, D, partition: BlockPartition) -> DevicePlan:
    """One device plan per (matrix, partition): the fp64 and fp32 instances
    of an adaptive policy share it."""
    cache = A.__dict__.setdefault("_plans", {})
    key = (partition.offsets.tobytes(), str(D.device))
    plan = cache.get(key)
    if plan is None:
        plan = DevicePlan(h, partition, A.row_ptr).bind(D)
        cache[key] = plan
    return plan


def setup(A: SparseMatrix, nb: int = 32, k: int = 2, t: int = 2,
          precision: Precision = Precision.F64,
          partition: BlockPartition | None = None) -> BjacPreconditioner:
    """Build a block-Jacobi preconditioner for square A (bjac.py:152-190).

    A's values are converted to the requested precision once, here, on the
    GPU.  Narrowing that overflows raises NarrowingOverflowError; a diagonal
    entry that is missing, zero, or underflows to zero is a ValueError naming
    the row.
    """
    if A.n != A.m:
        raise ValueError(f"matrix is {A.n}x{A.m}, preconditioner needs square")
    if partition is None:
        partition = BlockPartition.equal_split(A.n, nb)
    elif partition.n != A.n:
        raise ValueError(f"partition covers {partition.n} rows, matrix has {A.n}")
    if k < 1 or t < 1:
        raise ValueError("sweep counts k and t must be at least 1")
    return _setup_impl(A, k, t, precision, partition)


def _setup_impl(A: SparseMatrix, k: int, t: int, precision: Precision,
                partition: BlockPartition) -> BjacPreconditioner:
    """setup() after argument checks; also used for multi-GPU slabs, whose
    local matrix has ghost columns beyond its rows (distributed.py)."""
    torch = __import__("torch")
    h = _lib.Handle.get()
    D = A.device()
    # stored-diagonal presence, checked on the source values first
    src_vals = D.val64 if D.val64 is not None else D.val32
    f64src = D.val64 is not None
    dsrc = torch.empty(A.n, dtype=src_vals.dtype, device=D.device)
    missing, zero = C.c_int64(), C.c_int64()
    fn = h.lib.mpb_setup_diag_f64 if f64src else h.lib.mpb_setup_diag_f32
    _lib.check(fn(h.ptr, A.n, _lib.ptr(D.row_ptr), _lib.ptr(D.col_idx),
                  _lib.ptr(src_vals), _lib.ptr(dsrc), C.byref(missing),
                  C.byref(zero)), "setup")
    if missing.value >= 0:
        raise ValueError(f"row {int(missing.value)} has no stored diagonal entry")
    D, dvals = _device_values(A, precision, h)
    if (precision is Precision.F64) == f64src:
        ddiag, zrow = dsrc, int(zero.value)
    else:
        ddiag = torch.empty(A.n, dtype=dvals.dtype, device=D.device)
        z2 = C.c_int64()
        fn = h.lib.mpb_setup_diag_f64 if precision is Precision.F64 else h.lib.mpb_setup_diag_f32
        _lib.check(fn(h.ptr, A.n, _lib.ptr(D.row_ptr), _lib.ptr(D.col_idx),
                      _lib.ptr(dvals), _lib.ptr(ddiag), C.byref(missing),
                      C.byref(z2)), "setup")
        zrow = int(z2.value)
    if zrow >= 0:
        if float(dsrc[zrow].item()) != 0.0:
            raise ValueError(f"diagonal of row {zrow} underflows to zero in {precision}")
        raise ValueError(f"zero diagonal entry at row {zrow}")
    plan = _shared_plan(h, A, D, partition)
    return BjacPreconditioner(partition, int(k), int(t), precision, A, D,
                              dvals, ddiag, plan)


__all__ = ["BlockPartition", "BjacPreconditioner", "setup",
           "NarrowingOverflowError"]
