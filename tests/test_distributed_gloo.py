"""Multi-GPU host logic on the CPU, world size 2 over gloo.

Each rank takes its slab from paper_2407_15973_b200.distributed (slab
bounds at block boundaries, ghost renumbering, halo plan — the code the
NCCL path uses), then runs the distributed PCG with the oracle's arithmetic:
halos by gloo send/recv, dot products as per-rank device-order tree sums
all-reduced by gloo.  The result must equal, bit for bit, a single-process
solve that uses global kernels and the same rank-split dot order: any error
in the slab split, the renumbering or the halo plan would change x.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _system(name="c2", n=12):
    from paper_2407_15973_b200 import problems
    from paper_2407_15973_b200.bjac import BlockPartition
    cs = problems.make_config(name, n)
    return cs, BlockPartition.fixed_size(cs.A.n, cs.block_rows)


def _in_block(rp, ci, offsets, m):
    blk = np.searchsorted(offsets, np.arange(m), side="right") - 1
    rows = np.repeat(np.arange(m), np.diff(rp))
    c = ci.astype(np.int64)
    own = c < m
    cb = np.full(c.size, -1)
    cb[own] = blk[c[own]]
    return (own & (cb == blk[rows])).astype(np.uint8)


def _diag(rp, ci, vals, m):
    rows = np.repeat(np.arange(m), np.diff(rp))
    d = np.zeros(m, vals.dtype)
    hit = ci.astype(np.int64) == rows
    d[rows[hit]] = vals[hit]
    return d


class _Ops:
    """Local arithmetic of one slab (oracle kernels) + the exchange."""

    def __init__(self, O, slab, halo_fn, allreduce_fn):
        self.O, self.s = O, slab
        m = slab.m
        self.rp, self.ci = slab.row_ptr, slab.col_idx
        self.v64 = slab.values
        self.v32 = slab.values.astype(np.float32)
        self.inb = _in_block(self.rp, self.ci, slab.offsets, m)
        self.d64 = _diag(self.rp, self.ci, self.v64, m)
        self.d32 = _diag(self.rp, self.ci, self.v32, m)
        self.tiles, _ = O.plan_tiles(slab.offsets, self.rp)
        self.halo, self.allreduce = halo_fn, allreduce_fn

    def ext(self, v):
        out = np.zeros(self.s.m + self.s.ghosts, v.dtype)
        out[:self.s.m] = v
        self.halo(out)
        return out

    def matvec(self, vals, v):
        out = np.empty(self.s.m, vals.dtype)
        self.O.csr_matvec(self.rp, self.ci, vals, self.ext(v), out)
        return out

    def apply(self, r, low, k, t):
        vals, d = (self.v32, self.d32) if low else (self.v64, self.d64)
        dt = vals.dtype
        r = r.astype(dt)
        m = self.s.m
        z = np.empty(m, dt)
        tmp = np.empty(m, dt)
        self.O.block_jacobi_sweeps(self.rp, self.ci, vals, self.inb, d, t, r, z, tmp, 0, m)
        for _ in range(k - 1):
            az = self.matvec(vals, z)
            w = np.empty(m, dt)
            self.O.block_jacobi_sweeps(self.rp, self.ci, vals, self.inb, d, t, r - az, w, tmp, 0, m)
            z = z + w
        return z.astype(np.float64)

    def dot(self, a, b):
        return self.allreduce(self.O.tree_dot(self.tiles, a, b))


def _pcg(ops, b, kind, adp_tol, k, t, tol, cap):
    """solver.py:101-184 on one slab (x0 = 0)."""
    from paper_2407_15973_b200.policies import PolicyKind, choose_branch
    kind = PolicyKind(kind)
    x = np.zeros(b.size)
    r = b.copy()
    r0 = np.sqrt(ops.dot(r, r))
    relres, rho_prev, p, trace = 1.0, 0.0, None, []
    for it in range(1, cap + 1):
        low = choose_branch(kind, adp_tol, relres) == "low"
        z = ops.apply(r, low, k, t)
        rho = ops.dot(r, z)
        p = z.copy() if p is None else z + (rho / rho_prev) * p
        q = ops.matvec(ops.v64, p)
        alpha = rho / ops.dot(p, q)
        x = x + alpha * p
        r = r - alpha * q
        rho_prev = rho
        relres = np.sqrt(ops.dot(r, r)) / r0
        trace.append(relres)
        if relres <= tol:
            break
    return x, np.array(trace)


def _reference(Ox, cs, part, nranks, kind, adp_tol):
    """Single process: global matvec / BJAC kernels, dot products summed
    per slab in device tile-tree order and then over slabs in rank order."""
    from paper_2407_15973_b200 import distributed as D
    bounds = D.slab_bounds(part, nranks, cs.A.row_ptr)
    slabs = [D.extract_slab(cs.A.row_ptr, cs.A.col_idx, cs.A.values, part, bounds, r)
             for r in range(nranks)]
    # global kernels (row sums do not depend on the split), rank-split dots
    A = cs.A
    d64, d32, v32, inb = Ox.setup_arrays(A.row_ptr, A.col_idx, A.values, part.offsets)
    tiles = [Ox.plan_tiles(s.offsets, s.row_ptr)[0] for s in slabs]

    def dot(a, b):
        tot = 0.0
        for s, tl in zip(slabs, tiles):
            tot = tot + Ox.tree_dot(tl, a[s.lo:s.hi], b[s.lo:s.hi])
        return tot

    class G:
        pass
    g = G()
    g.dot = dot
    g.v64 = A.values

    def matvec(vals, v):
        out = np.empty(A.n, vals.dtype)
        Ox.csr_matvec(A.row_ptr, A.col_idx, vals, v.astype(vals.dtype), out)
        return out
    g.matvec = matvec

    def apply(r, low, k, t):
        vals, d = (v32, d32) if low else (A.values, d64)
        return Ox.bjac_apply(A.row_ptr, A.col_idx, vals, inb, d, k, t, r.astype(vals.dtype)).astype(np.float64)
    g.apply = apply
    return _pcg(g, cs.b, kind, adp_tol, cs.k, cs.t, cs.res_tol, 10 * A.n)


def _worker(rank, nranks, port, kind, adp_tol, outdir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    from oracle import oracle as O
    from paper_2407_15973_b200 import distributed as D
    cs, part = _system()
    bounds = D.slab_bounds(part, nranks, cs.A.row_ptr)
    s = D.extract_slab(cs.A.row_ptr, cs.A.col_idx, cs.A.values, part, bounds, rank)

    def halo(vec):  # fill ghosts [m, m+ng) following the slab's halo plan
        m = s.m
        t = torch.from_numpy(vec)
        reqs = []
        if s.rank_lo >= 0:
            if s.send_lo:
                reqs.append(dist.isend(t[:s.send_lo].clone(), s.rank_lo))
            if s.recv_lo:
                buf = torch.empty(s.recv_lo, dtype=t.dtype)
                reqs.append(("lo", dist.irecv(buf, s.rank_lo), buf))
        if s.rank_hi >= 0:
            if s.send_hi:
                reqs.append(dist.isend(t[m - s.send_hi:m].clone(), s.rank_hi))
            if s.recv_hi:
                buf = torch.empty(s.recv_hi, dtype=t.dtype)
                reqs.append(("hi", dist.irecv(buf, s.rank_hi), buf))
        for rq in reqs:
            if isinstance(rq, tuple):
                side, w, buf = rq
                w.wait()
                if side == "lo":
                    vec[m:m + s.recv_lo] = buf.numpy()
                else:
                    vec[m + s.recv_lo:m + s.recv_lo + s.recv_hi] = buf.numpy()
            else:
                rq.wait()

    def allreduce(v):
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())

    ops = _Ops(O, s, halo, allreduce)
    x, trace = _pcg(ops, cs.b[s.lo:s.hi], kind, adp_tol, cs.k, cs.t, cs.res_tol, 10 * cs.A.n)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), x=x, trace=trace, lo=s.lo, hi=s.hi,
             ghost_rows=s.ghost_rows())
    dist.destroy_process_group()


def test_slab_bounds_and_ghosts():
    from paper_2407_15973_b200 import distributed as D
    cs, part = _system("c2", 16)
    for nranks in (1, 2, 3, 4, 8):
        bounds = D.slab_bounds(part, nranks, cs.A.row_ptr)
        assert bounds[0][0] == 0 and bounds[-1][1] == cs.A.n
        assert all(a[1] == b[0] for a, b in zip(bounds, bounds[1:]))
        assert all(lo % 64 == 0 for lo, _ in bounds)          # whole blocks
        for r in range(nranks):
            s = D.extract_slab(cs.A.row_ptr, cs.A.col_idx, cs.A.values, part, bounds, r)
            # ghosts: one z-plane each way for the 7-point stencil
            assert s.recv_lo == (256 if r > 0 else 0) and s.recv_hi == (256 if r < nranks - 1 else 0)
            # renumbered columns map back to the global ones, order kept
            g = np.concatenate((s.ghost_rows(), [-1]))
            loc = s.col_idx.astype(np.int64)
            glob = np.where(loc < s.m, loc + s.lo, g[np.clip(loc - s.m, 0, g.size - 1)])
            e0, e1 = cs.A.row_ptr[s.lo], cs.A.row_ptr[s.hi]
            np.testing.assert_array_equal(glob, cs.A.col_idx[e0:e1])
            if r > 0:
                prev = D.extract_slab(cs.A.row_ptr, cs.A.col_idx, cs.A.values, part, bounds, r - 1)
                assert s.send_lo == prev.recv_hi
    with pytest.raises(ValueError):
        D.slab_bounds(part, part.num_blocks + 1)


@pytest.mark.parametrize("kind,adp_tol", [("fixed-low", None), ("adaptive-hl", 1e-3)])
def test_two_rank_solve_matches_rank_split_reference(tmp_path, kind, adp_tol):
    from oracle import oracle as O
    O.build()
    nranks = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, nranks, port, kind, adp_tol, str(tmp_path)))
             for r in range(nranks)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    cs, part = _system()
    x_ref, tr_ref = _reference(O, cs, part, nranks, kind, adp_tol)
    x = np.zeros(cs.A.n)
    for r in range(nranks):
        z = np.load(tmp_path / f"rank{r}.npz")
        x[int(z["lo"]):int(z["hi"])] = z["x"]
        np.testing.assert_array_equal(z["trace"], tr_ref)
    np.testing.assert_array_equal(x, x_ref)
    # and the rank-split order changes iterations by no more than the band
    full = O.pcg_solve(cs.A.row_ptr, cs.A.col_idx, cs.A.values, cs.b, part.offsets, kind=kind,
                       adp_tol=adp_tol, k=cs.k, t=cs.t, res_tol=cs.res_tol, order="device")
    assert abs(full["iterations"] - tr_ref.size) <= 2


def _ovf_worker(rank, nranks, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    from paper_2407_15973_b200.distributed import global_first_overflow
    # rank 0 owns rows [0, 100) without an overflow; rank 1 owns [100, 250)
    # and overflowed at its local row 7 (value 1e300); rank 2 at local row 3
    lo = (0, 100, 250)[rank]
    local = (-1, 7, 3)[rank]
    val = (float("nan"), 1e300, -2e300)[rank]
    g, v = global_first_overflow(lo, local, val)
    np.save(os.path.join(out, f"ovf{rank}.npy"), np.array([g, v]))
    dist.destroy_process_group()


def test_global_first_overflow_three_ranks(tmp_path):
    """Multi-GPU narrowing overflow: every rank reports the globally first
    offending row and its value (ovf_first was rank-local)."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_ovf_worker, args=(r, 3, port, str(tmp_path))) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(3):
        g, v = np.load(tmp_path / f"ovf{r}.npy")
        assert int(g) == 107 and v == 1e300
