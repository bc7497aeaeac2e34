"""Multi-GPU PCG: z-slab row sharding, one process per GPU, NCCL over
NVLink/NVSwitch.

The global system is cut into contiguous row slabs at BJAC block
boundaries, so every block — and with it every inner Jacobi sweep — stays
on one GPU.  Each rank keeps its own rows 0..m-1 and renumbers the columns
it references outside the slab to ghost rows m.. (rows just below the slab,
owned by the previous rank, then rows just above, owned by the next one).
The stored entry order of every row (ascending global column) is kept, so
every row sum is bit-identical to the single-GPU kernels; only the dot
products change order (per-rank device-order sums, then an fp64 all-reduce).

Host logic here (slab bounds, local slab extraction, halo plans) is plain
numpy and is exercised by the gloo tests (tests/test_distributed_gloo.py);
the solve itself is ``mpb_pcg_solve_dist`` (NCCL send/recv halos and
all-reduces captured in the iteration graph).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bjac import BlockPartition


def slab_bounds(partition: BlockPartition, nranks: int, row_ptr=None) -> list:
    """Contiguous slabs [lo, hi) at block boundaries, balancing rows (or
    nonzeros when row_ptr is given).  Every rank gets at least one block."""
    offs = np.asarray(partition.offsets, np.int64)
    nb = offs.size - 1
    if nranks < 1 or nranks > nb:
        raise ValueError(f"cannot split {nb} blocks over {nranks} ranks")
    weight = offs if row_ptr is None else np.asarray(row_ptr, np.int64)[offs]
    total = weight[-1]
    cuts = [0]
    for r in range(1, nranks):
        target = total * r / nranks
        b = int(np.searchsorted(weight, target, side="left"))
        b = min(max(b, cuts[-1] + 1), nb - (nranks - r))
        cuts.append(b)
    cuts.append(nb)
    return [(int(offs[cuts[r]]), int(offs[cuts[r + 1]])) for r in range(nranks)]


def ghost_extent(row_ptr, col_idx, lo: int, hi: int):
    """(recv_lo, recv_hi): ghost rows below / above slab [lo, hi)."""
    row_ptr = np.asarray(row_ptr)
    cols = np.asarray(col_idx)[int(row_ptr[lo]):int(row_ptr[hi])]
    if cols.size == 0:
        return 0, 0
    return max(0, lo - int(cols.min())), max(0, int(cols.max()) + 1 - hi)


@dataclass
class Slab:
    """One rank's share of the system."""

    rank: int
    nranks: int
    lo: int
    hi: int
    row_ptr: np.ndarray      # local, int64, m+1
    col_idx: np.ndarray      # local numbering (own 0..m-1, ghosts m..)
    values: np.ndarray
    offsets: np.ndarray      # local block offsets (0..m)
    recv_lo: int
    recv_hi: int
    send_lo: int             # own rows sent down (= previous rank's recv_hi)
    send_hi: int             # own rows sent up (= next rank's recv_lo)

    @property
    def m(self) -> int:
        return self.hi - self.lo

    @property
    def ghosts(self) -> int:
        return self.recv_lo + self.recv_hi

    @property
    def rank_lo(self) -> int:
        return self.rank - 1 if self.rank > 0 else -1

    @property
    def rank_hi(self) -> int:
        return self.rank + 1 if self.rank + 1 < self.nranks else -1

    def ghost_rows(self) -> np.ndarray:
        """Global row of every ghost index m, m+1, ... (for checks)."""
        below = np.arange(self.lo - self.recv_lo, self.lo)
        above = np.arange(self.hi, self.hi + self.recv_hi)
        return np.concatenate((below, above))

    def halo(self) -> _lib.MpbHalo:
        h = _lib.MpbHalo()
        h.rank_lo, h.rank_hi = self.rank_lo, self.rank_hi
        h.recv_lo, h.recv_hi = self.recv_lo, self.recv_hi
        h.send_lo, h.send_hi = self.send_lo, self.send_hi
        return h


def extract_slab(row_ptr, col_idx, values, partition: BlockPartition, bounds, rank: int) -> Slab:
    """The rank's rows with ghost-renumbered columns (entry order kept)."""
    row_ptr = np.asarray(row_ptr, np.int64)
    col_idx = np.asarray(col_idx)
    lo, hi = bounds[rank]
    nranks = len(bounds)
    recv_lo, recv_hi = ghost_extent(row_ptr, col_idx, lo, hi)
    if rank == 0 and recv_lo or rank == nranks - 1 and recv_hi:
        raise ValueError("matrix references rows outside the global range")
    if rank > 0 and recv_lo > bounds[rank - 1][1] - bounds[rank - 1][0]:
        raise ValueError(f"rank {rank}: halo of {recv_lo} rows is deeper than the slab below")
    if rank + 1 < nranks and recv_hi > bounds[rank + 1][1] - bounds[rank + 1][0]:
        raise ValueError(f"rank {rank}: halo of {recv_hi} rows is deeper than the slab above")
    e0, e1 = int(row_ptr[lo]), int(row_ptr[hi])
    m = hi - lo
    c = col_idx[e0:e1].astype(np.int64)
    loc = np.where(c < lo, m + (c - (lo - recv_lo)),
                   np.where(c >= hi, m + recv_lo + (c - hi), c - lo))
    send_lo = ghost_extent(row_ptr, col_idx, *bounds[rank - 1])[1] if rank > 0 else 0
    send_hi = ghost_extent(row_ptr, col_idx, *bounds[rank + 1])[0] if rank + 1 < nranks else 0
    offs = np.asarray(partition.offsets, np.int64)
    local_offs = offs[(offs >= lo) & (offs <= hi)] - lo
    return Slab(rank, nranks, lo, hi, row_ptr[lo:hi + 1] - e0, loc.astype(np.int32),
                np.asarray(values)[e0:e1], local_offs, recv_lo, recv_hi, send_lo, send_hi)


def global_first_overflow(lo: int, local_index: int, local_value: float):
    """(global row, value) of the first narrowing overflow over all ranks:
    a MIN all-reduce of the global row (ranks without a local overflow offer
    2^62), then the owner's value by a SUM all-reduce (the others add 0)."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend() == "nccl" else torch.device("cpu")
    none = 1 << 62
    g = lo + local_index if local_index >= 0 else none
    t = torch.tensor([g], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    gmin = int(t.item())
    mine = g == gmin and gmin != none
    v = torch.tensor([local_value if mine else 0.0], dtype=torch.float64, device=dev)
    dist.all_reduce(v, op=dist.ReduceOp.SUM)
    return (gmin if gmin != none else -1), float(v.item())


class SlabSolver:
    """Distributed drop-in for ``pcg_solve`` on one rank (one process per
    GPU; torch.distributed must be initialised — the NCCL unique id travels
    over it).  Every rank passes the same global system; each keeps only its
    slab on its GPU."""

    def __init__(self, A, partition: BlockPartition, policy, k: int = 2, t: int = 2,
                 rank: int | None = None, nranks: int | None = None, device=None):
        import torch
        import torch.distributed as dist
        from . import bjac
        from .policies import MixedPreconditioner
        from .sparse import SparseMatrix

        self.rank = dist.get_rank() if rank is None else rank
        self.nranks = dist.get_world_size() if nranks is None else nranks
        self.bounds = slab_bounds(partition, self.nranks, A.row_ptr)
        self.slab = extract_slab(A.row_ptr, A.col_idx, A.values, partition, self.bounds, self.rank)
        s = self.slab
        self.A_loc = SparseMatrix.trusted(s.m, s.m + s.ghosts, s.row_ptr, s.col_idx, s.values)
        part_loc = BlockPartition(s.offsets)
        p_high = bjac._setup_impl(self.A_loc, k, t, policy.work, part_loc) if policy.needs_high else None
        p_low = bjac._setup_impl(self.A_loc, k, t, policy.low, part_loc) if policy.needs_low else None
        self.mp = MixedPreconditioner(policy, p_high, p_low)
        self.h = _lib.Handle.get(device)
        uid = (C.c_char * 128)()
        if self.rank == 0:
            _lib.check(self.h.lib.mpb_comm_unique_id(uid), "mpb_comm_unique_id")
        box = [bytes(uid)]
        if self.nranks > 1:
            dist.broadcast_object_list(box, src=0)
        uid = (C.c_char * 128).from_buffer_copy(box[0])
        self.comm = C.c_void_p()
        _lib.check(self.h.lib.mpb_comm_create(self.h.ptr, self.rank, self.nranks, uid,
                                              C.byref(self.comm)), "mpb_comm_create")
        self._torch = torch

    def solve(self, b_local, config=None, x0_local=None):
        """Solve on this rank's slab; b_local: this slab's rows of b."""
        from .solver import SolveConfig, _run_solve
        config = config or SolveConfig()
        return _run_solve(self.A_loc, b_local, self.mp, config, x0_local,
                          dist=(self.comm, self.slab.halo(), self.slab.ghosts,
                                self._global_overflow),
                          n_global=self.bounds[-1][1])

    def _global_overflow(self, res) -> None:
        """After a narrowing overflow (the count is already global): every
        rank reports the globally first offending row and its value, as the
        one-GPU solve would (sparse.py:207-213).  res.overflow_index is the
        local row on the rank that saw an overflow itself, else -1."""
        g, v = global_first_overflow(self.slab.lo, int(res.overflow_index),
                                     float(res.err_value))
        res.overflow_index = g
        res.err_value = v

    def profile_iteration(self, config=None, branch: str = "low", reps: int = 20) -> dict:
        """Per-kernel times of one iteration on this slab (no communication)."""
        from .solver import SolveConfig, profile_iteration
        config = config or SolveConfig()
        return profile_iteration(self.A_loc, self.mp, config=config, branch=branch, reps=reps,
                                 ghosts=self.slab.ghosts, n_global=self.bounds[-1][1])

    def __del__(self):
        try:
            if self.comm:
                self.h.lib.mpb_comm_destroy(self.comm)
        except Exception:  # interpreter shutdown
            pass


class LocalSlabGroup:
    """Every slab of a multi-GPU solve on ONE GPU, in one process: one
    private handle, one in-process comm (mpb_comm_create_local) and one host
    thread per slab, each running ``mpb_pcg_solve_dist`` on its slab.  The
    library's in-process group replaces NCCL: all ranks' work goes to one
    stream, and at each halo exchange / all-reduce the ranks meet at a host
    barrier while rank 0 enqueues the copies and a rank-ordered sum.  It runs
    the multi-GPU code path (slab plans, ghost columns, halos, all-reduced
    scalar steps) with more ranks than GPUs; the arithmetic is the NCCL
    path's (a two-rank sum is exact in either order)."""

    def __init__(self, A, partition: BlockPartition, policy, nranks: int, k: int = 2, t: int = 2,
                 device=None):
        import threading
        import torch
        from . import bjac
        from .policies import MixedPreconditioner
        from .sparse import SparseMatrix

        self.device = torch.cuda.current_device() if device is None else int(device)
        self.nranks = int(nranks)
        self.n = int(A.n)
        self.bounds = slab_bounds(partition, self.nranks, A.row_ptr)
        self.slabs = [extract_slab(A.row_ptr, A.col_idx, A.values, partition, self.bounds, r)
                      for r in range(self.nranks)]
        self.A_loc, self.mp = [], []
        for s in self.slabs:
            Al = SparseMatrix.trusted(s.m, s.m + s.ghosts, s.row_ptr, s.col_idx, s.values)
            part = BlockPartition(s.offsets)
            ph = bjac._setup_impl(Al, k, t, policy.work, part) if policy.needs_high else None
            pl = bjac._setup_impl(Al, k, t, policy.low, part) if policy.needs_low else None
            self.A_loc.append(Al)
            self.mp.append(MixedPreconditioner(policy, ph, pl))
        L = _lib.load()
        self._L = L
        self.group = C.c_void_p()
        _lib.check(L.mpb_local_group_create(self.device, self.nranks, C.byref(self.group)),
                   "mpb_local_group_create")
        # every rank (its handle and its thread's torch copies) works on the
        # group's one stream: nothing orders through the legacy default stream
        self.stream_ptr = int(L.mpb_local_group_stream(self.group) or 0)
        self.stream = torch.cuda.ExternalStream(self.stream_ptr, device=self.device)
        torch.cuda.current_stream(self.device).synchronize()  # setup work (default stream) done
        self.comms, self.handles = [], []
        for r in range(self.nranks):
            c = C.c_void_p()
            _lib.check(L.mpb_comm_create_local(self.group, r, C.byref(c)), "mpb_comm_create_local")
            self.comms.append(c)
            self.handles.append(_lib.Handle(self.device, stream=self.stream_ptr))
        self._ovf = {}
        self._ovf_barrier = threading.Barrier(self.nranks)
        # the device structures (SELL packing, plan layouts) are built here,
        # once, on the calling thread: the rank threads only solve
        from .solver import _dev_struct
        for Al, m in zip(self.A_loc, self.mp):
            _dev_struct(Al, m)
        torch.cuda.current_stream(self.device).synchronize()

    def _overflow_hook(self, rank):
        def hook(res):
            # every rank saw the same global count; the first offending row
            # over all ranks, as global_first_overflow does over NCCL
            idx = int(res.overflow_index)
            self._ovf[rank] = (self.slabs[rank].lo + idx if idx >= 0 else None, float(res.err_value))
            self._ovf_barrier.wait()
            hits = [v for v in self._ovf.values() if v[0] is not None]
            g, v = min(hits) if hits else (-1, float("nan"))
            res.overflow_index = g
            res.err_value = v
            self._ovf_barrier.wait()
        return hook

    def solve(self, b, config=None, x0=None):
        """Solve with the global right-hand side b (host array); returns
        (global x as a host array, the per-rank SolveReports)."""
        import threading
        import numpy as _np
        from .solver import SolveConfig, _run_solve
        config = config or SolveConfig()
        b = _np.asarray(b, _np.float64)
        reps, errs = [None] * self.nranks, [None] * self.nranks

        torch = __import__("torch")

        def run(r):
            s = self.slabs[r]
            try:
                with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
                    reps[r] = _run_solve(
                    self.A_loc[r], _np.ascontiguousarray(b[s.lo:s.hi]), self.mp[r], config,
                    None if x0 is None else _np.ascontiguousarray(_np.asarray(x0)[s.lo:s.hi]),
                    dist=(self.comms[r], s.halo(), s.ghosts, self._overflow_hook(r)),
                    n_global=self.n, handle=self.handles[r])
                    self.stream.synchronize()
            except BaseException as e:  # re-raised in the caller's thread
                errs[r] = e

        th = [threading.Thread(target=run, args=(r,)) for r in range(self.nranks)]
        for t_ in th:
            t_.start()
        for t_ in th:
            t_.join()
        for e in errs:
            if e is not None:
                raise e
        x = _np.concatenate([_np.asarray(rep.x) for rep in reps])
        return x, reps

    def close(self):
        """Release the ranks' handles, comms and the group (in that order:
        the handles use the group's stream)."""
        try:
            if not getattr(self, "group", None):
                return  # closed already (the group's stream no longer exists)
            if getattr(self, "stream", None) is not None:
                self.stream.synchronize()
            for h in getattr(self, "handles", []):
                if h.ptr:
                    self._L.mpb_destroy(h.ptr)
                    h.ptr = C.c_void_p()
            self.handles = []
            for c in getattr(self, "comms", []):
                self._L.mpb_comm_destroy(c)
            self.comms = []
            self.stream = None
            self._L.mpb_local_group_destroy(self.group)
            self.group = None
        except Exception:  # interpreter shutdown
            pass

    def __del__(self):
        self.close()
