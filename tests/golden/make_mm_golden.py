"""Matrix Market fixtures: a handful of files exercising the format's corners
(symmetric expansion, duplicates, Fortran exponents, comments, blank lines)
and the CSR the reference's mm_read makes of each, plus the reference's
error class/message prefix for malformed files.

Run in the build container (the reference is not on the GPU box):
    python tests/golden/make_mm_golden.py
It imports the reference package read-only from /root/reference/pkg/src and
writes tests/golden/mm_golden.npz (files are stored as text inside it).
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

GOOD = {
    "general": "%%MatrixMarket matrix coordinate real general\n% c\n3 3 4\n1 1 4.0\n2 2 5.5\n3 3 2\n1 3 -1.25\n",
    "symmetric": ("%%MatrixMarket matrix coordinate real symmetric\n\n4 4 6\n1 1 10\n2 1 -1\n2 2 9\n"
                  "3 2 -2.5D-01\n4 3 -1d0\n4 4 8.0\n"),
    "duplicates": "%%MatrixMarket matrix coordinate real general\n2 2 5\n1 1 1\n1 1 2\n2 2 3\n2 1 0.5\n2 1 0.25\n",
    "empty_rows": "%%MatrixMarket matrix coordinate real general\n4 4 2\n4 4 1.0\n1 1 2.0\n",
    "banner_case": "%%MatrixMarket MATRIX Coordinate REAL General\n1 1 1\n1 1 3.0e+00\n",
}
BAD = {
    "no_banner": "matrix coordinate real general\n1 1 1\n1 1 1\n",
    "array": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n",
    "sym_rect": "%%MatrixMarket matrix coordinate real symmetric\n2 3 0\n",
    "short_size": "%%MatrixMarket matrix coordinate real general\n2 2\n",
    "bad_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "bad_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n",
    "too_many": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 2\n",
    "too_few": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n",
    "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
}


def main():
    from mpcg import mmio
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, text in GOOD.items():
            p = os.path.join(tmp, name + ".mtx")
            open(p, "w").write(text)
            A = mmio.mm_read(p)
            out[f"good/{name}/text"] = np.array(text)
            out[f"good/{name}/shape"] = np.array([A.n, A.m])
            out[f"good/{name}/row_ptr"] = np.asarray(A.row_ptr, np.int64)
            out[f"good/{name}/col_idx"] = np.asarray(A.col_idx, np.int64)
            out[f"good/{name}/values"] = np.asarray(A.values, np.float64)
        for name, text in BAD.items():
            p = os.path.join(tmp, name + ".mtx")
            open(p, "w").write(text)
            try:
                mmio.mm_read(p)
                raise SystemExit(f"{name}: the reference accepted it")
            except mmio.MatrixMarketError as e:
                out[f"bad/{name}/text"] = np.array(text)
                out[f"bad/{name}/message"] = np.array(str(e).replace(p, "<path>"))
    np.savez(os.path.join(HERE, "mm_golden.npz"), **out)
    print(f"wrote {len(GOOD)} good and {len(BAD)} bad cases")


if __name__ == "__main__":
    main()
