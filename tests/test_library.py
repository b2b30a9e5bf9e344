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


def test_stats_struct_matches_header():
    """ipdg_stats as declared in include/ipdg.h: int64, 2 doubles, 2 int32, double = 40 bytes."""
    import ctypes
    import re
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ipdg.h")).read()
    body = re.search(r"typedef struct \{(.*?)\} ipdg_stats;", hdr, re.S).group(1)
    fields = re.findall(r"^\s*(int64_t|double|int32_t)\s+(\w+);", body, re.M)
    assert [n for _, n in fields] == [n for n, _ in _lib.ipdg_stats._fields_]
    assert ctypes.sizeof(_lib.ipdg_stats) == 40


def test_tangential_face_derivative_identity():
    """The k_tpb face-derivative split (sipdg_tpb.cuh) rests on: the derivative of u ALONG face f at its
    nodes depends only on the face values (the nodal basis functions of the other nodes vanish on the
    face, so their tangential derivative there is zero), via one 1-D matrix D1D for all three faces
    (face 0: d/dr, face 1: d/ds - d/dr, face 2: d/ds, face nodes in ascending order).  Checked on the
    oracle's reference element for every degree."""
    for N in range(1, 9):
        ref = RefElem(N)
        F = ref.Fmask
        D1D = ref.Dr[np.ix_(F[0], F[0])]
        for f, T in ((0, ref.Dr), (1, ref.Ds - ref.Dr), (2, ref.Ds)):
            rows = T[F[f]]
            want = np.zeros_like(rows)
            want[:, F[f]] = D1D
            assert np.abs(rows - want).max() <= 1e-10 * np.abs(ref.Dr).max(), (N, f)
