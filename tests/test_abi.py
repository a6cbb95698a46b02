"""CPU-only checks of the C ABI: the library loads, exports every declared
symbol, and host-side validation returns the documented status codes (these
paths return before any CUDA call)."""
import ctypes
import os

import numpy as np
import pytest

import paper_1802_10291_b200 as mci

pytestmark = pytest.mark.skipif(not os.path.exists(mci.LIB_PATH), reason="libmci.so not built")


def test_exports_every_header_symbol():
    lib = ctypes.CDLL(mci.LIB_PATH)
    names = mci.header_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n


def test_version_and_status_strings():
    assert "sm_100a" in mci.version()
    lib = mci._lib_handle()
    for s in range(8):
        assert lib.mci_status_str(s)


def _create(M, N, L, bank, dtype=0, flags=0, null=()):
    lib = mci._lib_handle()
    arr, keep = mci._systems(bank)
    h = ctypes.c_void_p()
    nb = np.asarray(list(null), dtype=np.int64)
    st = lib.mci_plan_create(ctypes.byref(h), M, N, L, ctypes.addressof(arr),
                             nb.ctypes.data if len(nb) else None, len(nb), dtype, flags)
    return st, h


def test_alias_band_size_errors():
    f = [("identity",), ("derivative", 1)]
    assert _create(2, 32, 32, f)[0] == mci.MCI_E_ALIAS          # L < MN
    assert _create(2, 32, 80, f)[0] == mci.MCI_E_ALIAS          # L not a multiple of N
    assert _create(2, 24, 36, f)[0] == mci.MCI_E_ALIAS          # arbitrary-length path: L < MN
    assert _create(2, 24, 60, f)[0] == mci.MCI_E_ALIAS          # arbitrary-length path: L % N != 0
    assert _create(1, 1, 16, [("identity",)])[0] == mci.MCI_E_SIZE
    assert _create(2, 40000, 160000, f)[0] == mci.MCI_E_SIZE    # exceeds the arbitrary-length path
    assert _create(3, 1, 16, [("identity",)] * 3)[0] in (mci.MCI_E_SIZE, mci.MCI_E_BAND)
    assert _create(0, 32, 256, f)[0] == mci.MCI_E_ARG
    assert _create(2, 32, 256, f, dtype=7)[0] == mci.MCI_E_ARG
    st, h = _create(2, 32, 256, f, flags=16)
    assert st == mci.MCI_E_ARG and not h.value


def test_singular_bin_reported():
    """Example 3: M = 1 Hilbert channel is singular at n = 0."""
    st, h = _create(1, 16, 64, [("hilbert",)])
    assert st == mci.MCI_E_SINGULAR and not h.value
    assert mci._lib_handle().mci_last_singular_bin() == 0
    # two identical channels: singular everywhere; the first class built is q = 0
    st, _ = _create(2, 16, 64, [("identity",), ("identity",)])
    assert st == mci.MCI_E_SINGULAR


def test_non_hermitian_table_rejected():
    M, N = 1, 16
    tab = np.ones(M * N, dtype=complex)
    tab[3] = 2.0  # breaks b(-k) = conj b(k)
    st, _ = _create(1, 16, 64, [("table", tab)])
    assert st == mci.MCI_E_UNSUPPORTED


def test_execute_argument_checks_without_plan():
    lib = mci._lib_handle()
    assert lib.mci_execute_1d(None, 1, None, None, None, None) == mci.MCI_E_ARG
    assert lib.mci_execute_2d(None, 1, None, None, None) == mci.MCI_E_ARG
    assert lib.mci_plan_launches(None, 4) == 0
    lib.mci_plan_destroy(None)
