"""DG gradient G^e and divergence D^e with central fluxes (oracle; test infrastructure only).

SURVEY NEXT-2.  Eqs. INS_SD_4_1 / INS_SD_4_2:

  (v, G^e p)_E = (v, grad p)_E + 1/2 (v, n [[p]])_dE
  (v, D^e u)_E = (v, div u)_E  + 1/2 (v, n . [[u]])_dE

with the paper's jump [[w]] = w+ - w- (P:85).  Boundary conditions: along velocity-Dirichlet
boundaries u* = g_D and p* = p-, along velocity-Neumann (outflow) boundaries u* = u- and p* = 0;
homogeneous data, imposed by mirroring the exterior trace (u* = {u}, p* = {p}).  One mesh serves the
pressure Poisson solve and these operators, so the face codes are read as PRESSURE boundary types
(reading R20): code 1 (pressure Dirichlet = velocity outflow): p+ = -p-, u+ = u-;
code 2 (pressure Neumann = velocity Dirichlet): p+ = p-, u+ = -u-.

Assembled by quadrature from the variational forms, like oracle.assemble (no derivative or lift
matrices, no trace maps): returns the weak matrices (v_i, G_x p) etc.; the nodal operators are
(J^e M)^{-1} times them, block by block.  A second, independent route (nodal_grad_lift) applies the
strong form with the lift operator, G p = grad p + 1/2 sum_f (sJ/J) LIFT_f n [[p]].
"""
import numpy as np
import scipy.sparse as sp

from . import meshops
from .assemble import _basis_phys, _to_reference
from .quadrature import line_rule, triangle_rule

P_MIRROR = {1: -1.0, 2: 1.0}  # p+ = s p- on boundary faces by code (pressure Dirichlet / Neumann)
U_MIRROR = {1: 1.0, 2: -1.0}  # u+ = s u-


def weak_derivative(VX, VY, EToV, bc, ref, axis, mirror):
    """CSR matrix W with (W w)_{e,i} = (l_i, d_axis w)_E + 1/2 (l_i, n_axis [[w]])_dE, exterior traces
    from the face neighbour on interior faces and w+ = mirror[code] w- on boundary faces."""
    N, Np = ref.N, ref.Np
    K = EToV.shape[0]
    geo = meshops.affine_geometry(VX, VY, EToV)
    nx, ny, sJ = meshops.face_geometry(VX, VY, EToV)
    EToE, _, _, _ = meshops.connectivity(VX, VY, EToV, bc, ref)
    nrm = nx if axis == 0 else ny
    rows, cols, vals = [], [], []
    dofs = np.arange(K)[:, None] * Np + np.arange(Np)[None, :]
    # volume: J sum_q w_q l_i d_axis l_j
    rq, sq, wq = triangle_rule(N + 1)
    V = ref.eval_basis(rq, sq)
    Pr, Ps = ref.eval_grad_basis(rq, sq)
    G = geo["Ginv"]  # [[rx, ry], [sx, sy]]
    Pd = G[:, 0, axis][:, None, None] * Pr[None] + G[:, 1, axis][:, None, None] * Ps[None]
    Ve = geo["J"][:, None, None] * np.einsum("q,qi,eqj->eij", wq, V, Pd)
    rows.append(np.repeat(dofs, Np, axis=1).ravel())
    cols.append(np.tile(dofs, (1, Np)).ravel())
    vals.append(Ve.ravel())
    # faces of every element (the form is per element, not symmetric)
    tq, wt = line_rule(N + 1)
    for f in range(3):
        e = np.arange(K)
        a = EToV[e, f]
        b = EToV[e, (f + 1) % 3]
        px = VX[a][:, None] + (tq[None, :] + 1) / 2 * (VX[b] - VX[a])[:, None]
        py = VY[a][:, None] + (tq[None, :] + 1) / 2 * (VY[b] - VY[a])[:, None]
        W = 0.5 * wt[None, :] * sJ[e, f][:, None] * nrm[e, f][:, None]
        r, s = _to_reference(geo["Jm"], VX[EToV[:, 0]], VY[EToV[:, 0]], px, py)
        Vm, _, _ = _basis_phys(ref, geo, e, r, s)
        code = bc[:, f]
        # -1/2 (l_i, n w-) from every face; the exterior part below
        selfc = np.where(code == 0, -1.0, 0.0)
        for c, sgn in mirror.items():
            selfc = np.where(code == c, sgn - 1.0, selfc)
        B = selfc[:, None, None] * np.einsum("eq,eqi,eqj->eij", W, Vm, Vm)
        rows.append(np.repeat(dofs, Np, axis=1).ravel())
        cols.append(np.tile(dofs, (1, Np)).ravel())
        vals.append(B.ravel())
        inter = np.nonzero(code == 0)[0]
        if inter.size:
            eP = EToE[inter, f]
            rp, sp_ = _to_reference(geo["Jm"][eP], VX[EToV[eP, 0]], VY[EToV[eP, 0]], px[inter], py[inter])
            Vp, _, _ = _basis_phys(ref, geo, eP, rp, sp_)
            Bp = np.einsum("eq,eqi,eqj->eij", W[inter], Vm[inter], Vp)
            rows.append(np.repeat(dofs[inter], Np, axis=1).ravel())
            cols.append(np.tile(dofs[eP], (1, Np)).ravel())
            vals.append(Bp.ravel())
    n = K * Np
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsr()


def _inverse_mass(VX, VY, EToV, ref, w):
    J = meshops.affine_geometry(VX, VY, EToV)["J"]
    Wr = np.asarray(w, dtype=np.float64).reshape(-1, ref.Np)
    return (np.linalg.solve(ref.M, Wr.T).T / J[:, None]).reshape(-1, ref.Np)


def dg_grad(VX, VY, EToV, bc, ref, p):
    """Nodal G p (Eq. INS_SD_4_1): returns (Gx p, Gy p), each K x Np."""
    p = np.asarray(p, dtype=np.float64).ravel()
    gx = weak_derivative(VX, VY, EToV, bc, ref, 0, P_MIRROR) @ p
    gy = weak_derivative(VX, VY, EToV, bc, ref, 1, P_MIRROR) @ p
    return _inverse_mass(VX, VY, EToV, ref, gx), _inverse_mass(VX, VY, EToV, ref, gy)


def dg_div(VX, VY, EToV, bc, ref, ux, uy):
    """Nodal D u (Eq. INS_SD_4_2), K x Np."""
    ux = np.asarray(ux, dtype=np.float64).ravel()
    uy = np.asarray(uy, dtype=np.float64).ravel()
    w = (weak_derivative(VX, VY, EToV, bc, ref, 0, U_MIRROR) @ ux
         + weak_derivative(VX, VY, EToV, bc, ref, 1, U_MIRROR) @ uy)
    return _inverse_mass(VX, VY, EToV, ref, w)


def nodal_grad_lift(VX, VY, EToV, bc, ref, p):
    """Second route for G p: strong form with the lift (Eq. elLift): grad p at the nodes from
    Dr, Ds plus 1/2 sum_f (sJ/J) LIFT_f (n [[p]]) with traces through Fmask and coordinate-matched
    neighbour nodes (oracle.meshops.connectivity)."""
    Np, Nfp = ref.Np, ref.N + 1
    P = np.asarray(p, dtype=np.float64).reshape(-1, Np)
    geo = meshops.affine_geometry(VX, VY, EToV)
    nx, ny, sJ = meshops.face_geometry(VX, VY, EToV)
    _, _, vmapM, vmapP = meshops.connectivity(VX, VY, EToV, bc, ref)
    pr, ps = P @ ref.Dr.T, P @ ref.Ds.T
    gx = geo["rx"][:, None] * pr + geo["sx"][:, None] * ps
    gy = geo["ry"][:, None] * pr + geo["sy"][:, None] * ps
    flat = P.ravel()
    pm = flat[vmapM].reshape(-1, 3, Nfp)
    pp = flat[vmapP].reshape(-1, 3, Nfp)
    for c, sgn in P_MIRROR.items():
        m = (bc == c)[:, :, None]
        pp = np.where(m, sgn * pm, pp)
    jump = pp - pm
    F = (sJ / geo["J"][:, None])[:, :, None]
    lx = (F * nx[:, :, None] * jump).reshape(-1, 3 * Nfp) @ ref.LIFT.T
    ly = (F * ny[:, :, None] * jump).reshape(-1, 3 * Nfp) @ ref.LIFT.T
    return gx + 0.5 * lx, gy + 0.5 * ly
