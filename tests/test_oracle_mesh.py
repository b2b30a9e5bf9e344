"""Pins for the oracle's connectivity, affine geometry and penalty (CPU only)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import meshops
from oracle.refelem import RefElem
from paper_1801_00246_b200 import meshgen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_geometry_example():
    g = GOLD["geometry_example"]
    v = np.array(g["vertices"], dtype=float)
    geo = meshops.affine_geometry(v[:, 0], v[:, 1], np.array([[0, 1, 2]]))
    for k in ("J", "rx", "sy", "ry", "sx"):
        assert abs(geo[k][0] - g[k]) < 1e-15


def test_tau_example():
    g = GOLD["tau_example"]
    # shared edge (0,0)-(0,1) of length 1; right triangle area 0.25 (h- = 0.25), left area 0.5 (h+ = 0.5)
    VX = np.array([0.0, 0.0, 0.5, -1.0])
    VY = np.array([0.0, 1.0, 0.0, 0.0])
    EToV = np.array([[0, 2, 1], [0, 1, 3]])
    bc = np.array([[1, 1, 0], [0, 1, 1]])
    ref = RefElem(g["N"])
    geo = meshops.affine_geometry(VX, VY, EToV)
    _, _, sJ = meshops.face_geometry(VX, VY, EToV)
    EToE, EToF, _, _ = meshops.connectivity(VX, VY, EToV, bc, ref)
    tau = meshops.penalty(g["N"], geo, sJ, EToE, EToF)
    assert abs(geo["area"][0] - 0.25) < 1e-15 and abs(geo["area"][1] - 0.5) < 1e-15
    assert abs(tau[0, 2] - g["tau"]) < 1e-13 and abs(tau[1, 0] - g["tau"]) < 1e-13


def test_c1_closed_forms():
    """C1 (4x4 cells, '/' diagonals): J = 1/64, 1/h = 8 on legs and 8 sqrt2 on diagonals, tau = 6/h."""
    m = meshgen.square(4)
    geo = meshops.affine_geometry(m["VX"], m["VY"], m["EToV"])
    nx, ny, sJ = meshops.face_geometry(m["VX"], m["VY"], m["EToV"])
    EToE, EToF, _, _ = meshops.connectivity(m["VX"], m["VY"], m["EToV"], m["bc"], RefElem(2))
    tau = meshops.penalty(2, geo, sJ, EToE, EToF)
    assert np.allclose(geo["J"], 1 / 64, atol=1e-16)
    F = sJ / geo["J"][:, None]
    diag = np.isclose(2 * sJ, math.sqrt(2) / 4)
    assert np.allclose(F[~diag], 8) and np.allclose(F[diag], 8 * math.sqrt(2))
    assert np.allclose(tau[~diag], 48) and np.allclose(tau[diag], 48 * math.sqrt(2))


@pytest.mark.parametrize("seed", [0, 1])
def test_mesh_invariants(seed):
    m = meshgen.square(9, jitter=0.2, diag="random", order="random", seed=seed)
    ref = RefElem(3)
    VX, VY, EToV = m["VX"], m["VY"], m["EToV"]
    geo = meshops.affine_geometry(VX, VY, EToV)
    assert abs(geo["area"].sum() - 1.0) < 1e-12  # sum_e 2 J_e = |Omega|
    assert np.all(geo["J"] > 0)
    # G^e is the inverse of the affine Jacobian
    prod = np.einsum("eij,ejk->eik", geo["Ginv"], geo["Jm"])
    assert np.abs(prod - np.eye(2)).max() < 1e-12
    nx, ny, sJ = meshops.face_geometry(VX, VY, EToV)
    assert np.allclose(nx ** 2 + ny ** 2, 1, atol=1e-14)
    EToE, EToF, vmapM, vmapP = meshops.connectivity(VX, VY, EToV, m["bc"], ref)
    inner = EToE >= 0
    e2, f2 = EToE[inner], EToF[inner]
    assert np.allclose(nx[inner], -nx[e2, f2], atol=1e-13) and np.allclose(ny[inner], -ny[e2, f2], atol=1e-13)
    assert np.allclose(sJ[inner], sJ[e2, f2], atol=1e-15)
    # involutive trace pairing with coincident coordinates
    x, y = meshops.physical_nodes(VX, VY, EToV, ref)
    xf, yf = x.ravel(), y.ravel()
    assert np.abs(xf[vmapM] - xf[vmapP]).max() < 1e-12 and np.abs(yf[vmapM] - yf[vmapP]).max() < 1e-12
    for e, f in zip(*np.nonzero(inner)):
        e2, f2 = EToE[e, f], EToF[e, f]
        for k in range(ref.Nfp):
            k2 = int(np.nonzero(vmapM[e2, f2] == vmapP[e, f, k])[0][0])
            assert vmapP[e2, f2, k2] == vmapM[e, f, k]
    # every boundary face carries a code, interior faces none
    assert np.all((m["bc"] == 0) == inner)


def test_connectivity_rejects_bad_mesh():
    m = meshgen.square(2)
    bc = m["bc"].copy()
    bc[0, np.nonzero(bc[0] == 0)[0][0]] = 1  # boundary tag on an interior face
    with pytest.raises(ValueError):
        meshops.connectivity(m["VX"], m["VY"], m["EToV"], bc, RefElem(1))
    EToV = m["EToV"].copy()
    EToV[0] = EToV[0, ::-1]  # clockwise element
    with pytest.raises(ValueError):
        meshops.affine_geometry(m["VX"], m["VY"], EToV)
