"""Matrix Market ingestion against fixtures made by the
reference's own mm_read (tests/golden/make_mm_golden.py): same CSR for the
format's corner cases, same error messages for malformed files."""
import os

import numpy as np
import pytest

from conftest import ROOT, random_spd_csr

FIX = np.load(os.path.join(ROOT, "tests", "golden", "mm_golden.npz"))


def _cases(kind):
    return sorted({k.split("/")[1] for k in FIX.files if k.startswith(kind + "/")})


@pytest.mark.parametrize("name", _cases("good"))
def test_mm_read_matches_reference(tmp_path, name):
    from paper_2407_15973_b200.mmio import mm_read
    p = tmp_path / f"{name}.mtx"
    p.write_text(str(FIX[f"good/{name}/text"]))
    A = mm_read(p)
    assert [A.n, A.m] == list(FIX[f"good/{name}/shape"])
    np.testing.assert_array_equal(A.row_ptr, FIX[f"good/{name}/row_ptr"])
    np.testing.assert_array_equal(A.col_idx, FIX[f"good/{name}/col_idx"])
    np.testing.assert_array_equal(A.values, FIX[f"good/{name}/values"])


@pytest.mark.parametrize("name", _cases("bad"))
def test_mm_read_errors_match_reference(tmp_path, name):
    from paper_2407_15973_b200.mmio import MatrixMarketError, mm_read
    p = tmp_path / f"{name}.mtx"
    p.write_text(str(FIX[f"bad/{name}/text"]))
    with pytest.raises(MatrixMarketError) as e:
        mm_read(p)
    assert str(e.value) == str(FIX[f"bad/{name}/message"])


def test_mm_round_trip_is_exact(tmp_path):
    from paper_2407_15973_b200.mmio import mm_read, mm_write
    rng = np.random.default_rng(3)
    A = random_spd_csr(200, 0.05, rng)
    A.values[:5] = [1e-300, -2.5e300, np.pi, 1 / 3, 0.1]
    mm_write(A, tmp_path / "a.mtx", comment="two\nlines")
    B = mm_read(tmp_path / "a.mtx")
    np.testing.assert_array_equal(B.row_ptr, A.row_ptr)
    np.testing.assert_array_equal(B.col_idx, A.col_idx)
    np.testing.assert_array_equal(B.values, A.values)
