"""Matrix Market coordinate I/O (reference: pkg/src/mpcg/mmio.py:38-143).

SURVEY §8(f) 4: external SPD matrices into the solver.  Same contract as the
reference: coordinate format, real field, general or symmetric symmetry,
1-based indices, '%' comments, Fortran 'D' exponents; symmetric files are
expanded (off-diagonal entries mirrored) and duplicates summed
(SparseMatrix.from_coo); anything else raises MatrixMarketError.  The body
is parsed in bulk with numpy (one vectorised pass), falling back to a
line-by-line scan only to name the offending line of a malformed file.
Writing emits coordinate real general, row-major, values as repr() (the
shortest string that round-trips the float64).
"""
from __future__ import annotations

import numpy as np

from .sparse import SparseMatrix

BANNER = "%%MatrixMarket"


class MatrixMarketError(ValueError):
    """Malformed or unsupported Matrix Market content."""


def _value(token: str, lineno: int) -> float:
    try:
        return float(token)
    except ValueError:
        try:
            return float(token.lower().replace("d", "e"))
        except ValueError:
            raise MatrixMarketError(f"line {lineno}: bad numeric value {token!r}") from None


def _header(line: str) -> str:
    if not line.startswith(BANNER):
        raise MatrixMarketError("missing %%MatrixMarket banner")
    f = line.split()
    if len(f) != 5:
        raise MatrixMarketError(f"banner has {len(f)} fields, expected 5")
    obj, fmt, field, sym = (t.lower() for t in f[1:])
    if obj != "matrix":
        raise MatrixMarketError(f"unsupported object {obj!r}")
    if fmt != "coordinate":
        raise MatrixMarketError(f"unsupported format {fmt!r}, only coordinate is handled")
    if field != "real":
        raise MatrixMarketError(f"unsupported field {field!r}, only real is handled")
    if sym not in ("general", "symmetric"):
        raise MatrixMarketError(f"unsupported symmetry {sym!r}")
    return sym


def _scan(body, first_lineno, n, m, nnz):
    """Line-by-line parse (diagnostics path): rows, cols, vals."""
    rows = np.empty(nnz, np.int64)
    cols = np.empty(nnz, np.int64)
    vals = np.empty(nnz, np.float64)
    k = 0
    for off, line in enumerate(body):
        lineno = first_lineno + off
        s = line.strip()
        if not s or s.startswith("%"):
            continue
        if k >= nnz:
            raise MatrixMarketError(f"line {lineno}: more entries than the declared {nnz}")
        t = s.split()
        if len(t) != 3:
            raise MatrixMarketError(f"line {lineno}: entry needs 'row col value'")
        try:
            i, j = int(t[0]), int(t[1])
        except ValueError:
            raise MatrixMarketError(f"line {lineno}: non-integer index") from None
        if not (1 <= i <= n and 1 <= j <= m):
            raise MatrixMarketError(f"line {lineno}: index ({i}, {j}) outside {n}x{m}")
        rows[k], cols[k], vals[k] = i - 1, j - 1, _value(t[2], lineno)
        k += 1
    if k != nnz:
        raise MatrixMarketError(f"file declares {nnz} entries but contains {k}")
    return rows, cols, vals


def mm_read(path) -> SparseMatrix:
    """A Matrix Market file as a float64 SparseMatrix."""
    with open(path, "r", encoding="ascii", errors="replace") as fh:
        text = fh.read().split("\n")
    sym = _header(text[0] if text else "")
    k = 1
    while k < len(text) and (not text[k].strip() or text[k].strip().startswith("%")):
        k += 1
    if k >= len(text):
        raise MatrixMarketError("missing size line")
    size = text[k].split()
    if len(size) != 3:
        raise MatrixMarketError(f"line {k + 1}: size line needs 'rows cols nnz'")
    try:
        n, m, nnz = (int(t) for t in size)
    except ValueError:
        raise MatrixMarketError(f"line {k + 1}: non-integer size field") from None
    if min(n, m, nnz) < 0:
        raise MatrixMarketError(f"line {k + 1}: negative size field")
    if sym == "symmetric" and n != m:
        raise MatrixMarketError("symmetric matrix must be square")
    body = text[k + 1:]
    entries = [s for s in (ln.strip() for ln in body) if s and not s.startswith("%")]
    try:  # bulk path: well-formed files parse in one vectorised pass
        if len(entries) != nnz:
            raise ValueError
        tok = np.array(" ".join(entries).split(), dtype=object)
        if tok.size != 3 * nnz:
            raise ValueError
        tok = tok.reshape(nnz, 3) if nnz else tok.reshape(0, 3)
        rows = tok[:, 0].astype(np.int64) - 1
        cols = tok[:, 1].astype(np.int64) - 1
        vals = tok[:, 2].astype(np.float64)
        if nnz and (rows.min() < 0 or rows.max() >= n or cols.min() < 0 or cols.max() >= m):
            raise ValueError
    except (ValueError, TypeError):
        rows, cols, vals = _scan(body, k + 2, n, m, nnz)
    if sym == "symmetric":
        off = rows != cols
        rows, cols, vals = (np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                            np.concatenate([vals, vals[off]]))
    return SparseMatrix.from_coo(n, m, rows, cols, vals)


def mm_write(A: SparseMatrix, path, comment=None) -> None:
    """A SparseMatrix as coordinate real general, 1-based, row-major."""
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr)) + 1
    cols = A.col_idx.astype(np.int64) + 1
    vals = A.values.astype(np.float64)
    with open(path, "w", encoding="ascii") as fh:
        fh.write(f"{BANNER} matrix coordinate real general\n")
        for line in (str(comment).splitlines() if comment else []):
            fh.write(f"% {line}\n")
        fh.write(f"{A.n} {A.m} {A.nnz}\n")
        step = 1 << 20
        for lo in range(0, A.nnz, step):
            fh.writelines(f"{i} {j} {v!r}\n" for i, j, v in
                          zip(rows[lo:lo + step].tolist(), cols[lo:lo + step].tolist(),
                              vals[lo:lo + step].tolist()))
