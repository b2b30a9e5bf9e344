"""CPU checks of the C-ABI library: it loads, exports every symbol include/ipdg.h declares, and its
host-side setup (reference operators, built in C++ independently of oracle/) matches the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle.refelem import RefElem
from paper_1801_00246_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ipdg.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ipdg_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # the Python binding covers the same names
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)


def test_strerror_and_bad_degree():
    L = _lib.lib()
    assert L.ipdg_strerror(_lib.IPDG_EDEGREE).decode().startswith("degree")
    ctx = ctypes.c_void_p()
    assert L.ipdg_create(ctypes.byref(ctx), 9, 0) == _lib.IPDG_EDEGREE
    assert L.ipdg_create(ctypes.byref(ctx), 0, 0) == _lib.IPDG_EDEGREE
    assert L.ipdg_create(None, 2, 0) == _lib.IPDG_EINVAL
    buf = np.zeros(4)
    assert L.ipdg_refop_host(2, 99, buf.ctypes.data, 4) == _lib.IPDG_EINVAL


@pytest.mark.parametrize("N", range(1, 9))
def test_host_refops_match_oracle(N):
    """Setup parity: libipdg's C++ reference element == the oracle's, element by element."""
    L = _lib.lib()
    ref = RefElem(N)
    Np, Nfp = ref.Np, ref.Nfp

    def get(name, n):
        buf = np.zeros(n)
        assert L.ipdg_refop_host(N, _lib.OPS[name], buf.ctypes.data, n) == n
        return buf

    assert np.abs(get("r", Np) - ref.r).max() < 1e-14
    assert np.abs(get("s", Np) - ref.s).max() < 1e-14
    assert np.abs(get("Dr", Np * Np).reshape(Np, Np) - ref.Dr).max() < 1e-12 * max(1, np.abs(ref.Dr).max())
    assert np.abs(get("Ds", Np * Np).reshape(Np, Np) - ref.Ds).max() < 1e-12 * max(1, np.abs(ref.Ds).max())
    assert np.abs(get("M", Np * Np).reshape(Np, Np) - ref.M).max() < 1e-14
    assert np.abs(get("M1D", Nfp * Nfp).reshape(Nfp, Nfp) - ref.M1D).max() < 1e-14
    assert np.abs(get("LIFT", Np * 3 * Nfp).reshape(Np, 3 * Nfp) - ref.LIFT).max() < 1e-11 * np.abs(ref.LIFT).max()
    assert np.array_equal(get("Fmask", 3 * Nfp).reshape(3, Nfp).astype(int), ref.Fmask)
