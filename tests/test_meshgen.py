"""The synthetic workload generators (BASELINE configs C1-C5 shapes) produce valid meshes (CPU)."""
import numpy as np
import pytest

from oracle import meshops
from oracle.refelem import RefElem
from paper_1801_00246_b200 import meshgen, partition


def _valid(m):
    geo = meshops.affine_geometry(m["VX"], m["VY"], m["EToV"])  # raises on J <= 0
    EToE, _ = partition.global_connectivity(m["EToV"])
    assert np.all((EToE < 0) == (m["bc"] != 0))  # boundary codes exactly on boundary faces
    return geo


def test_c1_square():
    m = meshgen.square(4)
    geo = _valid(m)
    assert m["EToV"].shape[0] == 32 and np.allclose(geo["J"], 1 / 64)
    assert np.all(m["bc"][m["bc"] != 0] == meshgen.DIRICHLET)


@pytest.mark.parametrize("order", ["natural", "morton", "random"])
def test_c2_recipe_small(order):
    m = meshgen.square(20, jitter=0.2, diag="random", order=order, seed=2)
    geo = _valid(m)
    assert m["EToV"].shape[0] == 800 and abs(geo["area"].sum() - 1.0) < 1e-12


def test_morton_locality():
    m = meshgen.square(32, jitter=0.2, diag="random", order="morton", seed=2)
    EToE, _ = partition.global_connectivity(m["EToV"])
    e = np.arange(EToE.shape[0])[:, None]
    gap = np.abs(EToE - e)[EToE >= 0]
    assert np.median(gap) < 40  # neighbours are mostly close in the element order


def test_cylinder_small():
    m = meshgen.cylinder(h0=0.1, ratio=1.3)
    geo = _valid(m)
    area = (41.0 * 44.0) - 1.0
    assert abs(geo["area"].sum() - area) < 1e-9 * area
    a = m["EToV"][:, [0, 1, 2]]
    b = m["EToV"][:, [1, 2, 0]]
    xm = 0.5 * (m["VX"][a] + m["VX"][b])
    dirichlet = m["bc"] == meshgen.DIRICHLET
    assert np.all(np.abs(xm[dirichlet] - 25.0) < 1e-9)  # outflow only
    neu = m["bc"] == meshgen.NEUMANN
    ym = 0.5 * (m["VY"][a] + m["VY"][b])
    on_cyl = neu & (np.abs(xm) <= 0.5 + 1e-9) & (np.abs(ym) <= 0.5 + 1e-9)
    assert on_cyl.sum() > 0  # the cylinder wall is a Neumann boundary


def test_tiles_seams_and_parts():
    m, part = meshgen.tiles(6, 2, 2, seed=5)
    geo = _valid(m)
    assert m["EToV"].shape[0] == 4 * 72 and np.bincount(part).tolist() == [72] * 4
    assert abs(geo["area"].sum() - 4.0) < 1e-12
    ranks = partition.split(m, part, 4)
    assert partition.check_plan(ranks)
    MeshN = RefElem(2)
    meshops.connectivity(m["VX"], m["VY"], m["EToV"], m["bc"], MeshN)  # seams are conforming
