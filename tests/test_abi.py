"""The C-ABI library: loads without a GPU, exports every symbol the public
header declares, and its host-only entry points (status strings, the tile
plan) behave; the tile plan agrees with the oracle's restatement of
include/mpbjac_order.h."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "mpbjac.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mpb_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2407_15973_b200 import _lib
    return _lib.load()


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("mpb_pcg_solve", "mpb_bjac_apply_f32", "mpb_fmp_apply", "mpb_csr_matvec_f64",
                 "mpb_block_jacobi_sweeps_f64", "mpb_plan_create", "mpb_sell_create"):
        assert must in syms
    assert len(syms) >= 35


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert missing == []


def test_python_binding_covers_header():
    from paper_2407_15973_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_version_and_status_strings(lib):
    assert lib.mpb_version() >= 100
    assert lib.mpb_status_string(0) == b"ok"
    assert b"sweep" in lib.mpb_status_string(-4)
    assert b"SELL" in lib.mpb_status_string(-8)
    assert lib.mpb_status_string(-99) == b"unknown status"


def _plan_host(lib, offsets, row_ptr):
    offsets = np.ascontiguousarray(offsets, np.int64)
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    nb = offsets.size - 1
    out = np.empty(nb + int(offsets[-1]) // 256 + 2, np.int64)
    large = C.c_int()
    nt = lib.mpb_plan_tiles_host(nb, offsets.ctypes.data_as(C.c_void_p),
                                 row_ptr.ctypes.data_as(C.c_void_p),
                                 out.ctypes.data_as(C.c_void_p), C.byref(large))
    return out[:nt + 1], bool(large.value)


@pytest.mark.parametrize("case", ["r64", "r96", "nb32", "ragged", "dense"])
def test_tile_plan_matches_oracle(lib, oracle, case):
    rng = np.random.default_rng(5)
    n = 20000
    if case == "dense":
        lens = rng.integers(50, 200, n)
    else:
        lens = rng.integers(4, 8, n)
    row_ptr = np.concatenate(([0], np.cumsum(lens)))
    offsets = {"r64": np.append(np.arange(0, n, 64), n),
               "r96": np.append(np.arange(0, n, 96), n),
               "nb32": np.linspace(0, n, 33).astype(np.int64),
               "ragged": np.unique(np.concatenate(([0, n], rng.integers(1, n, 900)))),
               "dense": np.append(np.arange(0, n, 40), n)}[case]
    got, large = _plan_host(lib, offsets, row_ptr)
    want, wlarge = oracle.plan_tiles(offsets, row_ptr)
    np.testing.assert_array_equal(got, want)
    assert large == wlarge
    # tiles hold whole blocks unless a block is larger than a tile
    assert got[0] == 0 and got[-1] == n
    if not large:
        assert set(got.tolist()) <= set(offsets.tolist())
    assert np.all(np.diff(got) <= 256)


def test_tile_plan_rejects_bad_arguments(lib):
    assert lib.mpb_plan_tiles_host(0, None, None, None, None) < 0
