"""Test-system generators: the reference's 3-D diffusion families plus the
five benchmark configurations of BASELINE.json.

Setup-time host code (not the hot path).  The reference families
(const/ani/dis/rand, pkg/src/mpcg/problems.py:128-210) are restated here in
vectorised numpy and reproduce the reference's matrices bit for bit
(tests/test_problems.py pins that against golden fixtures).  Configs 2-5 have
no generator in the reference; they follow the recipe of SURVEY.md §8(d):

  U(s, m)   = splitmix64_stream(s, m)                 (problems.py:39-53)
  Nrm(s, m) = sqrt(-2 ln max(u[:m], 2^-53)) cos(2 pi u[m:]),  u = U(s, 2m)
  C1  kappa = 1, n=32,  b = 2 U(0,N) - 1, 64-row blocks, k=t=2, tol 1e-10
  C2  kappa = exp(2 Nrm(1,N)), n=128, b = U(1,N), fixed-low
  C3  kappa = 10^(-3+6 U(2,(n/8)^3)) on 8^3-cell blocks, n=256, b = U(2,N),
      adaptive-lh:1e-6
  C4  3-temperature system, n=128 cells, 3 unknowns per cell (cell-major),
      96-row blocks, b = U(3, 3n^3)
  C5  kappa = (1e-4 | 1e4 alternating every 16 z-planes) * exp(Nrm(4,N)),
      n=512, b = U(4,N), fixed-low, k=2, t=3, tol 1e-8

Grid ordering everywhere: node (i, j, k) -> row p = i + j n + k n^2, cell
arrays C-ordered [k, j, i]; h = 1/(n+1); face coefficient = harmonic mean
(2a)b/(a+b) of the two cells, a boundary face takes the cell's own value.

``device=True`` (make_config, diffusion_matrix, three_temperature,
splitmix64_stream) assembles the 7-point and 3-T operators and draws the
uniform streams on the GPU (mpb_assemble_stencil / mpb_expand_3t /
mpb_splitmix64_uniform: same IEEE operations, same
order, bit-identical; tests/test_gpu_parity.py pins it), which turns the
512^3 setup from minutes of numpy into a fraction of a second plus one
device-to-host copy.  Cell fields (kappa: exp/log/cos/pow) stay on the host,
where libm's correctly rounded results define them.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .sparse import SparseMatrix

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _gpu():
    from . import _lib
    return _lib.Handle.get()


def splitmix64_stream(seed: int, count: int, device: bool = False, a: float = 1.0,
                      b: float = 0.0) -> np.ndarray:
    """First `count` uniforms in [0,1) of the SplitMix64 stream for seed:
    state_i = seed + (i+1) gamma mod 2^64, mixed, top 53 bits scaled.
    device=True: drawn on the GPU (a*u + b, as a host array)."""
    if count < 0:
        raise ValueError("count must be nonnegative")
    if device:
        import torch
        from . import _lib
        h = _gpu()
        out = torch.empty(max(count, 1), dtype=torch.float64, device=f"cuda:{h.device}")
        _lib.check(h.lib.mpb_splitmix64_uniform(h.ptr, seed & ((1 << 64) - 1), count, float(a),
                                                float(b), _lib.ptr(out)), "splitmix64")
        return out[:count].cpu().numpy()
    out = np.empty(count, np.float64)
    chunk = 1 << 24
    s = np.uint64(seed & ((1 << 64) - 1))
    with np.errstate(over="ignore"):
        for lo in range(0, count, chunk):
            i = np.arange(lo + 1, min(count, lo + chunk) + 1, dtype=np.uint64)
            z = s + i * _GAMMA
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z ^= z >> np.uint64(31)
            out[lo:lo + i.size] = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return out


def normal_stream(seed: int, count: int) -> np.ndarray:
    """Box-Muller on two consecutive SplitMix64 blocks."""
    u = splitmix64_stream(seed, 2 * count)
    u1 = np.maximum(u[:count], 2.0 ** -53)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u[count:])


# ---------------------------------------------------------------------------
# 7-point finite-volume assembly
# ---------------------------------------------------------------------------

def _harmonic(a, b):
    return 2.0 * a * b / (a + b)


def face_arrays(kap3: np.ndarray, weights=(1.0, 1.0, 1.0)):
    """(xm, xp, ym, yp, zm, zp) per-cell face coefficients, flattened.
    Interior faces are computed once and shared by both neighbours, so the
    assembled matrix is symmetric bit for bit."""
    out = []
    for axis, w in ((2, weights[0]), (1, weights[1]), (0, weights[2])):
        n = kap3.shape[axis]
        a = np.take(kap3, np.arange(n - 1), axis=axis)
        b = np.take(kap3, np.arange(1, n), axis=axis)
        inner = w * _harmonic(a, b)
        fm = np.empty_like(kap3)
        fp = np.empty_like(kap3)
        sl = [slice(None)] * 3
        sl[axis] = slice(1, None)
        fm[tuple(sl)] = inner
        sl[axis] = 0
        fm[tuple(sl)] = w * np.take(kap3, 0, axis=axis)
        sl[axis] = slice(None, -1)
        fp[tuple(sl)] = inner
        sl[axis] = -1
        fp[tuple(sl)] = w * np.take(kap3, n - 1, axis=axis)
        out += [fm.ravel(), fp.ravel()]
    return out


def stencil_csr(n: int, faces, scale: float, extra_diag=None):
    """CSR arrays of the 7-point operator on an n^3 grid.

    Row entries in ascending column order zm, ym, xm, diag, xp, yp, zp;
    off-diagonals -(face*scale); diagonal ((((xm+xp)+ym)+yp)+zm)+zp)*scale
    (+ extra_diag).  Returns row_ptr int64, col_idx int32, values float64.
    """
    fxm, fxp, fym, fyp, fzm, fzp = faces
    N = n ** 3
    p = np.arange(N, dtype=np.int64)
    i = p % n
    j = (p // n) % n
    k = p // (n * n)
    has = [k > 0, j > 0, i > 0, None, i < n - 1, j < n - 1, k < n - 1]
    shift = [-n * n, -n, -1, 0, 1, n, n * n]
    face = [fzm, fym, fxm, None, fxp, fyp, fzp]
    cnt = np.ones(N, np.int64)
    for hm in has:
        if hm is not None:
            cnt += hm
    row_ptr = np.zeros(N + 1, np.int64)
    np.cumsum(cnt, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    pos = row_ptr[:-1].copy()
    for hm, sh, f in zip(has, shift, face):
        if hm is None:
            d = ((((fxm + fxp) + fym) + fyp) + fzm) + fzp
            d = d * scale
            if extra_diag is not None:
                d = d + extra_diag
            col[pos] = p
            val[pos] = d
            pos += 1
            continue
        sel = np.flatnonzero(hm)
        col[pos[sel]] = p[sel] + sh
        val[pos[sel]] = -(f[sel] * scale)
        pos[sel] += 1
    return row_ptr, col, val


# ---------------------------------------------------------------------------
# reference families (pkg/src/mpcg/problems.py:56-256)
# ---------------------------------------------------------------------------

class Family(enum.Enum):
    CONST = "const"
    ANI = "ani"
    DIS = "dis"
    RAND = "rand"


def family_kappa(n: int, family: Family, s: float = 1.0, seed: int = 0) -> np.ndarray:
    N = n ** 3
    if family in (Family.CONST, Family.ANI):
        return np.ones(N)
    if family is Family.DIS:
        x = (np.arange(n) + 1.0) / (n + 1)
        ins = (x >= 0.25) & (x <= 0.75)
        m = ins[:, None, None] & ins[None, :, None] & ins[None, None, :]
        return np.where(m, float(s), 1.0).ravel()
    return np.power(float(s), splitmix64_stream(seed, N))


def diffusion_matrix(n: int, kappa: np.ndarray, weights=(1.0, 1.0, 1.0),
                     validate: bool = True, device: bool = False) -> SparseMatrix:
    if device and n >= 2:
        return _diffusion_matrix_gpu(n, kappa, weights)
    kap3 = np.asarray(kappa, np.float64).reshape(n, n, n)
    row_ptr, col, val = stencil_csr(n, face_arrays(kap3, weights), float((n + 1) ** 2))
    N = n ** 3
    if validate:
        return SparseMatrix(N, N, row_ptr, col, val)
    return SparseMatrix.trusted(N, N, row_ptr, col, val)


def _diffusion_matrix_gpu(n: int, kappa, weights) -> SparseMatrix:
    """diffusion_matrix assembled on the GPU; the host copy is fetched once
    and the device CSR is kept as the matrix's GPU copy (no re-upload)."""
    import torch
    from . import _lib
    from .device import DeviceCSR, default_device
    h = _gpu()
    dev = default_device()
    N = n ** 3
    nnz = int(h.lib.mpb_stencil_nnz(n))
    kd = torch.from_numpy(np.ascontiguousarray(kappa, np.float64).ravel()).to(dev)
    rp = torch.empty(N + 1, dtype=torch.int32, device=dev)
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=torch.float64, device=dev)
    _lib.check(h.lib.mpb_assemble_stencil(h.ptr, n, _lib.ptr(kd), float(weights[0]), float(weights[1]),
                                          float(weights[2]), float((n + 1) ** 2), _lib.ptr(rp),
                                          _lib.ptr(col), _lib.ptr(val)), "assemble_stencil")
    rp_h = rp.cpu().numpy().astype(np.int64)
    A = SparseMatrix.trusted(N, N, rp_h, col.cpu().numpy(), val.cpu().numpy())
    A._dev[str(dev)] = DeviceCSR(N, N, rp, col, val64=val, host_row_ptr=rp_h)
    return A


def family_matrix(n: int, family: Family, s: float = 1.0, seed: int = 0) -> SparseMatrix:
    weights = (1.0, float(s), float(s)) if family is Family.ANI else (1.0, 1.0, 1.0)
    return diffusion_matrix(n, family_kappa(n, family, s, seed), weights)


def diag_augment(A: SparseMatrix, p_diag: float) -> SparseMatrix:
    """A with p_diag * (row's absolute sum, diagonal included) added to each
    diagonal entry (pkg/src/mpcg/problems.py:259-281): a preconditioner
    source of A's structure with other values.  The row sums use numpy's
    add.reduceat like the reference, so the result is bit-identical;
    p_diag = 0 gives a bitwise copy."""
    if p_diag < 0:
        raise ValueError("p_diag must be nonnegative")
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    diag_pos = np.flatnonzero(rows == A.col_idx)
    if diag_pos.size != A.n:
        have = np.zeros(A.n, dtype=bool)
        have[rows[diag_pos]] = True
        raise ValueError(f"row {int(np.flatnonzero(~have)[0])} has no stored diagonal entry")
    sums = np.zeros(A.n, dtype=A.values.dtype)
    nonempty = np.flatnonzero(np.diff(A.row_ptr) > 0)
    sums[nonempty] = np.add.reduceat(np.abs(A.values), A.row_ptr[nonempty])
    values = A.values.copy()
    values[diag_pos] = values[diag_pos] + A.values.dtype.type(p_diag) * sums
    return SparseMatrix(A.n, A.m, A.row_ptr, A.col_idx, values)


# ---------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------

@dataclass
class ConfigSystem:
    name: str
    A: SparseMatrix
    b: np.ndarray
    block_rows: int
    policies: tuple
    k: int
    t: int
    res_tol: float
    n: int
    note: str = ""


def kappa_c2(n: int) -> np.ndarray:
    return np.exp(2.0 * normal_stream(1, n ** 3))


def kappa_c3(n: int) -> np.ndarray:
    nb8 = n // 8
    v = 10.0 ** (-3.0 + 6.0 * splitmix64_stream(2, nb8 ** 3))
    c = np.arange(n) // 8
    idx = (c[:, None, None] * nb8 * nb8 + c[None, :, None] * nb8 + c[None, None, :])
    return v[idx].ravel()


def kappa_c5(n: int) -> np.ndarray:
    layer = np.where((np.arange(n) // 16) % 2 == 0, 1e-4, 1e4)
    base = np.broadcast_to(layer[:, None, None], (n, n, n)).ravel()
    return base * np.exp(normal_stream(4, n ** 3))


def three_temperature_fields(n: int):
    """Config 4's cell fields (host: libm's exp/sin/pow define them):
    D = T^3 and the exchange rates w_RE, w_EI."""
    N = n ** 3
    x = (np.arange(n) + 1.0) / (n + 1)
    sx = np.sin(2.0 * np.pi * x)
    smooth = sx[:, None, None] * sx[None, :, None] * sx[None, None, :]
    T = 0.01 + 9.99 * (0.5 + 0.5 * smooth)
    T = np.clip(T.ravel() * np.exp(0.1 * normal_stream(3, N)), 0.01, 10.0)
    D = T ** 3
    u = splitmix64_stream(103, 2 * N)
    w_re = 10.0 ** (-4.0 + 8.0 * u[:N])
    w_ei = 10.0 ** (-4.0 + 8.0 * u[N:])
    return D, w_re, w_ei


def _three_temperature_gpu(n: int) -> SparseMatrix:
    """three_temperature assembled on the GPU (mpb_assemble_stencil for the
    D operator, then mpb_expand_3t); the host copy is fetched once and the
    device CSR is kept as the matrix's GPU copy."""
    import torch
    from . import _lib
    from .device import DeviceCSR, default_device
    h = _gpu()
    dev = default_device()
    N = n ** 3
    D, w_re, w_ei = three_temperature_fields(n)
    scale = float((n + 1) ** 2)
    nnz1 = int(h.lib.mpb_stencil_nnz(n))
    f = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(dev)  # noqa: E731
    Dd, wr, we = f(D), f(w_re), f(w_ei)
    rp1 = torch.empty(N + 1, dtype=torch.int32, device=dev)
    c1 = torch.empty(nnz1, dtype=torch.int32, device=dev)
    v1 = torch.empty(nnz1, dtype=torch.float64, device=dev)
    _lib.check(h.lib.mpb_assemble_stencil(h.ptr, n, _lib.ptr(Dd), 1.0, 1.0, 1.0, scale, _lib.ptr(rp1),
                                          _lib.ptr(c1), _lib.ptr(v1)), "assemble_stencil")
    nnz = 3 * nnz1 + 4 * N
    rp = torch.empty(3 * N + 1, dtype=torch.int32, device=dev)
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=torch.float64, device=dev)
    _lib.check(h.lib.mpb_expand_3t(h.ptr, N, _lib.ptr(rp1), _lib.ptr(c1), _lib.ptr(v1), _lib.ptr(wr),
                                   _lib.ptr(we), 0.01 * scale, _lib.ptr(rp), _lib.ptr(col), _lib.ptr(val)),
               "expand_3t")
    del rp1, c1, v1
    rp_h = rp.cpu().numpy().astype(np.int64)
    A = SparseMatrix.trusted(3 * N, 3 * N, rp_h, col.cpu().numpy(), val.cpu().numpy())
    A._dev[str(dev)] = DeviceCSR(3 * N, 3 * N, rp, col, val64=val, host_row_ptr=rp_h)
    return A


def three_temperature(n: int, validate: bool = True, device: bool = False) -> SparseMatrix:
    """Config 4: per-component 7-point diffusion with D = T^3 plus per-cell
    radiation-electron (w_RE) and electron-ion (w_EI) exchange; unknown
    3 p + c (c = 0 radiation, 1 electron, 2 ion), cell-major.  device=True:
    assembled on the GPU (bit-identical)."""
    if device and n >= 2:
        return _three_temperature_gpu(n)
    N = n ** 3
    D, w_re, w_ei = three_temperature_fields(n)
    scale = float((n + 1) ** 2)
    rp1, col1, val1 = stencil_csr(n, face_arrays(D.reshape(n, n, n)), scale)
    cnt1 = np.diff(rp1)
    cells = np.arange(N, dtype=np.int64)
    rows1 = np.repeat(cells, cnt1)                  # cell of each stencil entry
    q = col1.astype(np.int64)                       # neighbour cell
    is_diag = q == rows1
    nlo = np.flatnonzero(is_diag) - rp1[:-1]        # stencil entries below the diagonal
    off = np.arange(col1.size, dtype=np.int64) - rp1[rows1]
    nlo_e = nlo[rows1]
    # row 3p+c: [lower stencil] [cell block: 3p+0..3p+2 couplings + diag] [upper stencil]
    cpl = (1, 2, 1)       # coupling entries per component
    dpos = (0, 1, 1)      # diagonal position inside the cell block
    cnt = (cnt1[:, None] + np.array(cpl)[None, :]).ravel()
    row_ptr = np.zeros(3 * N + 1, np.int64)
    np.cumsum(cnt, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    time_term = 0.01 * scale
    for c in range(3):
        base = row_ptr[3 * cells + c]
        slot = np.where(off < nlo_e, off,
                        np.where(is_diag, nlo_e + dpos[c], off + cpl[c]))
        dst = base[rows1] + slot
        col[dst] = 3 * q + c
        v = val1.copy()
        dd = v[is_diag] + time_term
        if c in (0, 1):
            dd = dd + w_re
        if c in (1, 2):
            dd = dd + w_ei
        v[is_diag] = dd
        val[dst] = v
        blk = base + nlo                             # first slot of the cell block
        if c == 0:
            col[blk + 1] = 3 * cells + 1
            val[blk + 1] = -w_re
        elif c == 1:
            col[blk] = 3 * cells
            val[blk] = -w_re
            col[blk + 2] = 3 * cells + 2
            val[blk + 2] = -w_ei
        else:
            col[blk] = 3 * cells + 1
            val[blk] = -w_ei
    if validate:
        return SparseMatrix(3 * N, 3 * N, row_ptr, col, val)
    return SparseMatrix.trusted(3 * N, 3 * N, row_ptr, col, val)


CONFIG_NAMES = ("c1", "c2", "c3", "c4", "c5")

#: grid size of each config at full scale (BASELINE.json configs[0..4])
FULL_N = {"c1": 32, "c2": 128, "c3": 256, "c4": 128, "c5": 512}


def make_config(name: str, n: int | None = None, validate: bool | None = None,
                device: bool = False) -> ConfigSystem:
    """Config name 'c1'..'c5' at its BASELINE.json size, or at grid size n
    (same recipe, for parity tests).  Same seeds, fields, blocks, policies.
    device=True: the operators (7-point and C4's 3-T) and right-hand
    sides built on the GPU (bit-identical)."""
    name = name.lower()
    if name in ("const128_nb32", "ani128_nb32"):
        # the reference's own acceptance problems (pkg/tests/test_acceptance.py:226-274) on its
        # default partition nb = 32 (bjac.py:152): 65,536-row blocks at n = 128, b = ones
        n = 128 if n is None else int(n)
        fam, scale = (Family.CONST, 1.0) if name.startswith("const") else (Family.ANI, 1000.0)
        A = family_matrix(n, fam, scale)
        if A.n % 32:
            raise ValueError("nb = 32 needs n^3 divisible by 32")
        return ConfigSystem(name, A, np.ones(A.n), A.n // 32, ("fixed-low", "uniform"), 2, 2, 1e-10, n,
                            f"{fam.value} family, b = ones, the reference's default partition nb = 32")
    n = FULL_N[name] if n is None else int(n)
    N = n ** 3
    if validate is None:
        validate = N <= 4_000_000
    if name == "c1":
        A = diffusion_matrix(n, np.ones(N), validate=validate, device=device)
        b = splitmix64_stream(0, N, device, 2.0, -1.0) if device else 2.0 * splitmix64_stream(0, N) - 1.0
        return ConfigSystem("c1", A, b, 64, ("uniform", "fixed-low"), 2, 2, 1e-10, n,
                            "3-D Poisson, 7-point, Dirichlet")
    if name == "c2":
        A = diffusion_matrix(n, kappa_c2(n), validate=validate, device=device)
        return ConfigSystem("c2", A, splitmix64_stream(1, N, device), 64, ("fixed-low",), 2, 2,
                            1e-10, n, "lognormal kappa, sigma=2")
    if name == "c3":
        if n % 8:
            raise ValueError("config 3 needs n divisible by 8")
        A = diffusion_matrix(n, kappa_c3(n), validate=validate, device=device)
        return ConfigSystem("c3", A, splitmix64_stream(2, N, device), 64, ("adaptive-lh:1e-6",),
                            2, 2, 1e-10, n, "8^3-cell blocks, kappa 1e-3..1e3")
    if name == "c4":
        A = three_temperature(n, validate=validate, device=device)
        return ConfigSystem("c4", A, splitmix64_stream(3, 3 * N, device), 96,
                            ("fixed-low", "adaptive-hl:10"), 2, 2, 1e-10, n,
                            "3-temperature radiation-diffusion stand-in")
    if name == "c5":
        A = diffusion_matrix(n, kappa_c5(n), validate=validate, device=device)
        return ConfigSystem("c5", A, splitmix64_stream(4, N, device), 64, ("fixed-low",), 2, 3,
                            1e-8, n, "layered multiscale kappa 1e-4/1e4")
    raise ValueError(f"unknown config {name!r}, expected one of {CONFIG_NAMES}")
