"""Mesh connectivity, affine geometry and the SIPDG penalty (oracle; test infrastructure only).

Inputs are the plain mesh arrays produced by ``paper_1801_00246_b200.meshgen``:
  VX, VY  (Nv,)  vertex coordinates
  EToV    (K,3)  counter-clockwise vertex ids
  bc      (K,3)  per element face: 0 interior, 1 Dirichlet, 2 Neumann
Face f of element e is the edge {EToV[e,f], EToV[e,(f+1)%3]} (faces 0,1,2 =
reference faces s=-1, r+s=0, r=-1; oracle.refelem).

Passages followed:
  P:49-53   -- neighbours share a face; n is the unit outward normal.
  P:462-487 (Eqs. operators1/2, elementOps) -- affine map x = Phi^e(r,s), its
            Jacobian G^e = [r_x s_x; r_y s_y], J^e = det, J^{ef} the face scaling
            (read as physical edge length / 2, reading R6).
  P:109-114 (Eq. Ch2.PenaltyParameter) -- tau = (N+1)(N+2)/2 max(1/h+, 1/h-),
            h = |E|/|dE^f|; on boundary faces h+ is undefined and tau uses h-
            only (reading R8).
"""
import numpy as np


def physical_nodes(VX, VY, EToV, ref):
    """Nodal coordinates x, y (K x Np): x = -(r+s)/2 x1 + (1+r)/2 x2 + (1+s)/2 x3 (Eq. operators1)."""
    v = EToV
    r, s = ref.r, ref.s
    x = 0.5 * (-np.outer(VX[v[:, 0]], r + s) + np.outer(VX[v[:, 1]], 1 + r) + np.outer(VX[v[:, 2]], 1 + s))
    y = 0.5 * (-np.outer(VY[v[:, 0]], r + s) + np.outer(VY[v[:, 1]], 1 + r) + np.outer(VY[v[:, 2]], 1 + s))
    return x, y


def affine_geometry(VX, VY, EToV):
    """Per element: Jacobian matrix entries and their inverse (Eq. operators2).

    Returns dict with xr, xs, yr, ys, J, rx, sx, ry, sy (each (K,)) and area.
    The inverse is taken with numpy.linalg.inv of the 2x2 Jacobian, element by element.
    """
    v = EToV
    x1, x2, x3 = VX[v[:, 0]], VX[v[:, 1]], VX[v[:, 2]]
    y1, y2, y3 = VY[v[:, 0]], VY[v[:, 1]], VY[v[:, 2]]
    xr, xs = (x2 - x1) / 2, (x3 - x1) / 2
    yr, ys = (y2 - y1) / 2, (y3 - y1) / 2
    Jm = np.stack([np.stack([xr, xs], -1), np.stack([yr, ys], -1)], -2)  # K x 2 x 2: d(x,y)/d(r,s)
    J = np.linalg.det(Jm)
    if np.any(J <= 0):
        raise ValueError("element %d has J <= 0" % int(np.nonzero(J <= 0)[0][0]))
    Ginv = np.linalg.inv(Jm)  # d(r,s)/d(x,y): [[rx, ry],[sx, sy]]
    return dict(xr=xr, xs=xs, yr=yr, ys=ys, J=J, rx=Ginv[:, 0, 0], ry=Ginv[:, 0, 1],
                sx=Ginv[:, 1, 0], sy=Ginv[:, 1, 1], area=2 * J, Jm=Jm, Ginv=Ginv)


def face_vertices(EToV, f):
    """(start, end) vertex ids of face f in counter-clockwise traversal."""
    return EToV[:, f], EToV[:, (f + 1) % 3]


def face_geometry(VX, VY, EToV):
    """Outward unit normals nx, ny and sJ (= edge length / 2), each (K, 3).

    The normal of a counter-clockwise edge a->b is (dy, -dx)/|d| with d = b - a.
    """
    K = EToV.shape[0]
    nx = np.zeros((K, 3))
    ny = np.zeros((K, 3))
    sJ = np.zeros((K, 3))
    for f in range(3):
        a, b = face_vertices(EToV, f)
        dx = VX[b] - VX[a]
        dy = VY[b] - VY[a]
        L = np.hypot(dx, dy)
        nx[:, f] = dy / L
        ny[:, f] = -dx / L
        sJ[:, f] = L / 2
    return nx, ny, sJ


def connectivity(VX, VY, EToV, bc, ref, tol=1e-10):
    """Face neighbours from a sorted-vertex-pair dictionary and node pairing by coordinates.

    Returns EToE, EToF (K x 3; -1 on boundary faces), vmapM, vmapP (K x 3 x Nfp global node
    ids; vmapP = vmapM on boundary faces).  Raises on a non-manifold edge, an interior-tagged
    face without neighbour, a boundary-tagged face with one, or unmatched trace nodes.
    """
    K = EToV.shape[0]
    Np, Nfp = ref.Np, ref.Nfp
    faces = {}
    for e in range(K):
        for f in range(3):
            key = tuple(sorted((int(EToV[e, f]), int(EToV[e, (f + 1) % 3]))))
            faces.setdefault(key, []).append((e, f))
    EToE = -np.ones((K, 3), dtype=np.int64)
    EToF = -np.ones((K, 3), dtype=np.int64)
    for key, lst in faces.items():
        if len(lst) > 2:
            raise ValueError("non-manifold edge %s" % (key,))
        if len(lst) == 2:
            (e1, f1), (e2, f2) = lst
            EToE[e1, f1], EToF[e1, f1] = e2, f2
            EToE[e2, f2], EToF[e2, f2] = e1, f1
    for e in range(K):
        for f in range(3):
            if bc[e, f] == 0 and EToE[e, f] < 0:
                raise ValueError("interior-tagged face (%d,%d) has no neighbour" % (e, f))
            if bc[e, f] != 0 and EToE[e, f] >= 0:
                raise ValueError("boundary-tagged face (%d,%d) has a neighbour" % (e, f))
    x, y = physical_nodes(VX, VY, EToV, ref)
    vmapM = np.zeros((K, 3, Nfp), dtype=np.int64)
    for f in range(3):
        vmapM[:, f, :] = np.arange(K)[:, None] * Np + ref.Fmask[f][None, :]
    vmapP = vmapM.copy()
    xf, yf = x.ravel(), y.ravel()
    _, _, sJ = face_geometry(VX, VY, EToV)
    ee, ff = np.nonzero(EToE >= 0)
    if ee.size:
        idM = vmapM[ee, ff]  # (n, Nfp)
        idP = vmapM[EToE[ee, ff], EToF[ee, ff]]
        D = (xf[idM][:, :, None] - xf[idP][:, None, :]) ** 2 + (yf[idM][:, :, None] - yf[idP][:, None, :]) ** 2
        j = np.argmin(D, axis=2)
        dmin = np.sqrt(np.take_along_axis(D, j[:, :, None], axis=2)[:, :, 0])
        bad = np.any(dmin > tol * 2 * sJ[ee, ff][:, None], axis=1)
        srt = np.sort(j, axis=1)
        bad |= np.any(srt[:, 1:] == srt[:, :-1], axis=1)
        if np.any(bad):
            k = int(np.nonzero(bad)[0][0])
            raise ValueError("trace nodes of face (%d,%d) do not match" % (ee[k], ff[k]))
        vmapP[ee, ff] = np.take_along_axis(idP, j, axis=1)
    return EToE, EToF, vmapM, vmapP


def penalty(N, geo, sJ, EToE, EToF):
    """tau (K x 3) by Eq. Ch2.PenaltyParameter: (N+1)(N+2)/2 * max(1/h-, 1/h+), h = |E|/|dE^f|."""
    c = (N + 1) * (N + 2) / 2.0
    area = geo["area"]
    length = 2 * sJ
    inv_h_minus = length / area[:, None]
    inv_h_plus = inv_h_minus.copy()
    inner = EToE >= 0
    inv_h_plus[inner] = length[inner] / area[EToE[inner]]
    return c * np.maximum(inv_h_minus, inv_h_plus)
