"""SIPDG bilinear form assembled by quadrature into a sparse matrix (oracle; test infrastructure only).

The positive operator A = -L + lambda (Eq. ellipticOp1) built from the
SIPDG Laplacian (Eq. INS_SD_5) with the penalty of Eq.
Ch2.PenaltyParameter, the paper's jump [[u]] = u+ - u-  and
average {u} = (u+ + u-)/2.  Summed over elements, the per-element form
of Eq. ellipticOp1 is the global symmetric form (R7):

  a(u,v) = sum_E [(grad u, grad v)_E + lambda (u,v)_E]
         - sum_{F interior} [({d_n u}, <v>)_F + ({d_n v}, <u>)_F - tau_F (<u>, <v>)_F]
         - sum_{F Dirichlet} [(d_n u, v)_F + (d_n v, u)_F - 2 tau_F (u, v)_F]

with <w> = w- - w+ (= -[[w]]) and n the outward normal of the "-" element.
Homogeneous boundary conditions by mirroring (R7): Dirichlet
u+ = -u-, grad u+ = grad u- (the 2 tau term); Neumann u+ = u-, grad u+ = -grad u-
(the face drops out).

This route uses no derivative matrices, lift matrices, Fmask or trace maps:
the nodal basis is evaluated directly at physical quadrature points through
the inverse affine map of each element (l_i = sum_k (V^{-T})_{ik} psi_k).
Quadrature is exact for the polynomial integrands (degree <= 2N).
"""
import numpy as np
import scipy.sparse as sp

from . import meshops
from .quadrature import line_rule, triangle_rule


def _to_reference(Jm, x1, y1, px, py):
    """(r, s) of physical points (K x nq) in elements with Jacobians Jm (K x 2 x 2)."""
    inv = np.linalg.inv(Jm)
    dx = px - x1[:, None]
    dy = py - y1[:, None]
    r = inv[:, 0, 0][:, None] * dx + inv[:, 0, 1][:, None] * dy - 1.0
    s = inv[:, 1, 0][:, None] * dx + inv[:, 1, 1][:, None] * dy - 1.0
    return r, s


def _basis_phys(ref, geo, elems, r, s):
    """Basis values and physical gradients of elements `elems` at reference points r,s (n x nq)."""
    n, nq = r.shape
    V = ref.eval_basis(r.ravel(), s.ravel()).reshape(n, nq, ref.Np)
    Pr, Ps = ref.eval_grad_basis(r.ravel(), s.ravel())
    Pr = Pr.reshape(n, nq, ref.Np)
    Ps = Ps.reshape(n, nq, ref.Np)
    G = geo["Ginv"][elems]  # [[rx, ry],[sx, sy]]
    Px = G[:, 0, 0][:, None, None] * Pr + G[:, 1, 0][:, None, None] * Ps
    Py = G[:, 0, 1][:, None, None] * Pr + G[:, 1, 1][:, None, None] * Ps
    return V, Px, Py


def assemble(VX, VY, EToV, bc, ref, lam=0.0, tau_scale=1.0):
    """Global SIPDG matrix (scipy CSR, size K*Np) of Eq. ellipticOp1 with homogeneous BCs."""
    N, Np = ref.N, ref.Np
    K = EToV.shape[0]
    geo = meshops.affine_geometry(VX, VY, EToV)
    nx, ny, sJ = meshops.face_geometry(VX, VY, EToV)
    EToE, EToF, _, _ = meshops.connectivity(VX, VY, EToV, bc, ref)
    tau = tau_scale * meshops.penalty(N, geo, sJ, EToE, EToF)
    rows, cols, vals = [], [], []

    # ---- volume: (grad phi_j, grad phi_i)_E + lambda (phi_j, phi_i)_E
    rq, sq, wq = triangle_rule(N + 1)
    V = ref.eval_basis(rq, sq)
    Pr, Ps = ref.eval_grad_basis(rq, sq)
    G = geo["Ginv"]
    Px = G[:, 0, 0][:, None, None] * Pr[None] + G[:, 1, 0][:, None, None] * Ps[None]
    Py = G[:, 0, 1][:, None, None] * Pr[None] + G[:, 1, 1][:, None, None] * Ps[None]
    Ke = np.einsum("q,eqi,eqj->eij", wq, Px, Px) + np.einsum("q,eqi,eqj->eij", wq, Py, Py)
    Ke += lam * np.einsum("q,qi,qj->ij", wq, V, V)[None]
    Ke *= geo["J"][:, None, None]
    dofs = np.arange(K)[:, None] * Np + np.arange(Np)[None, :]
    rows.append(np.repeat(dofs, Np, axis=1).ravel())
    cols.append(np.tile(dofs, (1, Np)).ravel())
    vals.append(Ke.ravel())

    # ---- faces
    tq, wt = line_rule(N + 1)
    eM, fM = [], []
    for e in range(K):
        for f in range(3):
            if bc[e, f] == 2:
                continue  # Neumann: no contribution
            if bc[e, f] == 0 and EToE[e, f] < e:
                continue  # interior face visited once, from its lower-numbered element
            eM.append(e)
            fM.append(f)
    eM = np.array(eM, dtype=np.int64)
    fM = np.array(fM, dtype=np.int64)
    if eM.size:
        a = EToV[eM, fM]
        b = EToV[eM, (fM + 1) % 3]
        px = VX[a][:, None] + (tq[None, :] + 1) / 2 * (VX[b] - VX[a])[:, None]
        py = VY[a][:, None] + (tq[None, :] + 1) / 2 * (VY[b] - VY[a])[:, None]
        W = wt[None, :] * sJ[eM, fM][:, None]  # physical weights
        n_x = nx[eM, fM][:, None, None]
        n_y = ny[eM, fM][:, None, None]
        v1 = EToV[eM, 0]
        r, s = _to_reference(geo["Jm"][eM], VX[v1], VY[v1], px, py)
        Vm, Pxm, Pym = _basis_phys(ref, geo, eM, r, s)
        DNm = n_x * Pxm + n_y * Pym
        t = tau[eM, fM]
        inter = bc[eM, fM] == 0
        dir_ = bc[eM, fM] == 1
        # Dirichlet faces: -(V^T W DN) - (DN^T W V) + 2 tau V^T W V
        if np.any(dir_):
            idx = np.nonzero(dir_)[0]
            Vd, Dd, Wd = Vm[idx], DNm[idx], W[idx]
            B = (-np.einsum("fq,fqi,fqj->fij", Wd, Vd, Dd) - np.einsum("fq,fqi,fqj->fij", Wd, Dd, Vd)
                 + 2 * t[idx][:, None, None] * np.einsum("fq,fqi,fqj->fij", Wd, Vd, Vd))
            d = dofs[eM[idx]]
            rows.append(np.repeat(d, Np, axis=1).ravel())
            cols.append(np.tile(d, (1, Np)).ravel())
            vals.append(B.ravel())
        if np.any(inter):
            idx = np.nonzero(inter)[0]
            eP = EToE[eM[idx], fM[idx]]
            v1p = EToV[eP, 0]
            rp, sp_ = _to_reference(geo["Jm"][eP], VX[v1p], VY[v1p], px[idx], py[idx])
            Vp, Pxp, Pyp = _basis_phys(ref, geo, eP, rp, sp_)
            DNp = n_x[idx] * Pxp + n_y[idx] * Pyp  # normal of the "-" element
            Jmp = np.concatenate([Vm[idx], -Vp], axis=2)  # <phi> = phi- - phi+
            Avg = 0.5 * np.concatenate([DNm[idx], DNp], axis=2)
            Wi = W[idx]
            B = (-np.einsum("fq,fqi,fqj->fij", Wi, Jmp, Avg) - np.einsum("fq,fqi,fqj->fij", Wi, Avg, Jmp)
                 + t[idx][:, None, None] * np.einsum("fq,fqi,fqj->fij", Wi, Jmp, Jmp))
            d = np.concatenate([dofs[eM[idx]], dofs[eP]], axis=1)
            n2 = 2 * Np
            rows.append(np.repeat(d, n2, axis=1).ravel())
            cols.append(np.tile(d, (1, n2)).ravel())
            vals.append(B.ravel())
    n = K * Np
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    return A.tocsr()


def mass_matrix(VX, VY, EToV, ref):
    """Block-diagonal global mass matrix J^e M (Eq. elementOps), assembled by quadrature."""
    K, Np, N = EToV.shape[0], ref.Np, ref.N
    geo = meshops.affine_geometry(VX, VY, EToV)
    rq, sq, wq = triangle_rule(N + 1)
    V = ref.eval_basis(rq, sq)
    Mref = np.einsum("q,qi,qj->ij", wq, V, V)
    blocks = geo["J"][:, None, None] * Mref[None]
    return sp.block_diag([b for b in blocks], format="csr")
