"""Matrix-free SIPDG action in primal form (oracle; test infrastructure only).

Same operator as oracle.assemble (Eq. ellipticOp1), written as a
numpy face loop over nodal traces instead of a quadrature assembly, so that
it can be timed at scale (bench.py cpu_baseline) and cross-checked against
the assembled matrix.  Per element e (paper jump [[u]] = u+ - u-):

  (v, A u)_E = (grad v, grad u)_E + lambda (v,u)_E
             + sum_f [ (v, -n.{grad u} - tau [[u]])_f + (n.grad v, 1/2 [[u]])_f ]

Volume:   J (Dx^T M Ux + Dy^T M Uy) + lambda J M u       (Eqs. elMass, elStiff, elementOps)
Face f:   (phi_i, g)_f = sJ (M1D g)  on the face-node rows (Lagrange basis
          of nodes off face f vanishes on f), and
          (n.grad phi_i, h)_f = sJ (Dn_f^T M1D h) with Dn_f the rows Fmask_f of
          n_x Dx + n_y Dy (the normal derivative is a degree-N polynomial,
          exactly represented at the N+1 face nodes).
Boundary mirroring (R7): Dirichlet u+ = -u-, grad u+ = grad u-;
Neumann u+ = u-, grad u+ = -grad u-.

It deliberately does NOT use the lift-into-q regrouping of the CUDA kernels
(Eq. ellipticOp3 style); only the textbook primal form above.
"""
import numpy as np

from . import meshops


class MFree:
    """Precomputed mesh data for the matrix-free oracle action."""

    def __init__(self, VX, VY, EToV, bc, ref, tau_scale=1.0):
        self.ref = ref
        self.K = EToV.shape[0]
        self.geo = meshops.affine_geometry(VX, VY, EToV)
        self.nx, self.ny, self.sJ = meshops.face_geometry(VX, VY, EToV)
        self.EToE, self.EToF, self.vmapM, self.vmapP = meshops.connectivity(VX, VY, EToV, bc, ref)
        self.tau = tau_scale * meshops.penalty(ref.N, self.geo, self.sJ, self.EToE, self.EToF)
        self.bc = np.asarray(bc)

    def apply(self, u, lam=0.0):
        ref, g = self.ref, self.geo
        K, Np = self.K, ref.Np
        U = np.asarray(u, dtype=np.float64).reshape(K, Np)
        rx, sx, ry, sy, J = g["rx"][:, None], g["sx"][:, None], g["ry"][:, None], g["sy"][:, None], g["J"][:, None]
        Ur = U @ ref.Dr.T
        Us = U @ ref.Ds.T
        Ux = rx * Ur + sx * Us
        Uy = ry * Ur + sy * Us
        # volume (grad v, grad u): J (Dx^T M Ux + Dy^T M Uy), Dx = rx Dr + sx Ds (row-vector form)
        MUx = Ux @ ref.M.T
        MUy = Uy @ ref.M.T
        out = J * (rx * (MUx @ ref.Dr) + sx * (MUx @ ref.Ds) + ry * (MUy @ ref.Dr) + sy * (MUy @ ref.Ds))
        if lam != 0.0:
            out = out + lam * J * (U @ ref.M.T)
        Uf, Uxf, Uyf = U.ravel(), Ux.ravel(), Uy.ravel()
        for f in range(3):
            idM = self.vmapM[:, f, :]
            idP = self.vmapP[:, f, :]
            nx = self.nx[:, f][:, None]
            ny = self.ny[:, f][:, None]
            um, up = Uf[idM], Uf[idP]
            dnm = nx * Uxf[idM] + ny * Uyf[idM]
            dnp = nx * Uxf[idP] + ny * Uyf[idP]
            code = self.bc[:, f][:, None]
            up = np.where(code == 1, -um, np.where(code == 2, um, up))
            dnp = np.where(code == 1, dnm, np.where(code == 2, -dnm, dnp))
            tau = self.tau[:, f][:, None]
            sJ = self.sJ[:, f][:, None]
            g1 = -0.5 * (dnm + dnp) + tau * (um - up)
            g2 = -0.5 * (um - up)
            Fm = ref.Fmask[f]
            out[:, Fm] += sJ * (g1 @ ref.M1D.T)
            h = sJ * (g2 @ ref.M1D.T)  # K x Nfp
            # Dn_f^T h with Dn_f = nx (rx Dr + sx Ds)[Fm] + ny (ry Dr + sy Ds)[Fm]
            ar = nx * rx + ny * ry
            as_ = nx * sx + ny * sy
            out += ar * (h @ ref.Dr[Fm, :]) + as_ * (h @ ref.Ds[Fm, :])
        return out
