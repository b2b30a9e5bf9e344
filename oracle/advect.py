"""Subcycling advection operator N~(U_bar, U~) (oracle; test infrastructure only).

SURVEY 8.6 row f4 (NEXT-4), PAPER.md Eq. INS_CUB_N:

  (v, N~^e)_E = -(grad v, F~(U_bar, U~))_E + (v, n . F~*)_dE,     F~ = U_bar (x) U~,

i.e. for each advected component c in {u~, v~}: the flux vector U_bar c, and the local Lax-Friedrichs
flux with Lambda = max(|n.U_bar-|, |n.U_bar+|) (Alg. SSS lambda_i).  The paper prints
F~* = {F~} + 1/2 n Lambda [[U~]] with [[w]] = w+ - w- (P:85), which is anti-dissipative; its Alg. SSS
 uses the dissipative sign, n.F~* = n.{F~} + 1/2 Lambda (c- - c+).  We follow Alg. SSS
(reading R27).  Boundary traces by mirroring with the velocity boundary types of reading R20
(R28): code 1 (pressure Dirichlet = outflow) U+ = U-, code 2 (velocity Dirichlet) U+ = -U-, applied to
both U_bar and U~.  The nodal output is N~^e = (J^e M)^{-1} times the weak form (Alg. SSV/SSS output N).

Computed by quadrature in PHYSICAL space, like oracle.assemble: the nodal basis is evaluated at the
quadrature points through the inverse affine map of each element (own and neighbour), no trace maps,
no lift or projection matrices.  The collapsed Gauss rule and the Gauss-Legendre face rule integrate the
degree-3N integrands exactly.
"""
import numpy as np

from . import meshops
from .assemble import _to_reference
from .quadrature import line_rule, triangle_rule

U_MIRROR = {1: 1.0, 2: -1.0}


def _npts(N):
    return (3 * N + 2) // 2 + 1  # 2 npts - 1 >= 3N


def advection(VX, VY, EToV, bc, ref, ub, vb, ut, vt):
    """Returns (Nu, Nv), each (K, Np): N~ applied to the advected components ut, vt (K, Np) with the
    advective velocity (ub, vb) (K, Np)."""
    N, Np = ref.N, ref.Np
    K = EToV.shape[0]
    geo = meshops.affine_geometry(VX, VY, EToV)
    nxf, nyf, sJ = meshops.face_geometry(VX, VY, EToV)
    EToE, _, _, _ = meshops.connectivity(VX, VY, EToV, bc, ref)
    J = geo["J"]
    # ---- volume: -(grad l_n, U_bar c)_E
    rq, sq, wq = triangle_rule(_npts(N))
    V = ref.eval_basis(rq, sq)                      # nq x Np
    Pr, Ps = ref.eval_grad_basis(rq, sq)
    G = geo["Ginv"]                                 # [[rx, ry], [sx, sy]]
    Px = G[:, 0, 0][:, None, None] * Pr[None] + G[:, 1, 0][:, None, None] * Ps[None]   # K x nq x Np
    Py = G[:, 0, 1][:, None, None] * Pr[None] + G[:, 1, 1][:, None, None] * Ps[None]
    ubq, vbq, utq, vtq = (f @ V.T for f in (ub, vb, ut, vt))                               # K x nq
    weak = np.zeros((2, K, Np))
    for c, cq in enumerate((utq, vtq)):
        weak[c] -= J[:, None] * np.einsum("q,eqn,eq->en", wq, Px, ubq * cq)
        weak[c] -= J[:, None] * np.einsum("q,eqn,eq->en", wq, Py, vbq * cq)
    # ---- faces: (l_n, n . F~*)_dE with the traces evaluated at physical points from both sides
    tq, wt = line_rule(_npts(N))
    e = np.arange(K)
    for f in range(3):
        a, b = EToV[e, f], EToV[e, (f + 1) % 3]
        px = VX[a][:, None] + (tq[None, :] + 1) / 2 * (VX[b] - VX[a])[:, None]
        py = VY[a][:, None] + (tq[None, :] + 1) / 2 * (VY[b] - VY[a])[:, None]
        r, s = _to_reference(geo["Jm"], VX[EToV[:, 0]], VY[EToV[:, 0]], px, py)
        Lm = ref.eval_basis(r.ravel(), s.ravel()).reshape(K, -1, Np)        # own basis at the points
        vals_m = [np.einsum("eqn,en->eq", Lm, fld) for fld in (ub, vb, ut, vt)]
        nb = EToE[e, f]
        inner = nb >= 0
        vals_p = [np.empty_like(v) for v in vals_m]
        if np.any(inner):
            ne = nb[inner]
            rp, sp_ = _to_reference(geo["Jm"][ne], VX[EToV[ne, 0]], VY[EToV[ne, 0]], px[inner], py[inner])
            Lp = ref.eval_basis(rp.ravel(), sp_.ravel()).reshape(ne.size, -1, Np)
            for vp, fld in zip(vals_p, (ub, vb, ut, vt)):
                vp[inner] = np.einsum("eqn,en->eq", Lp, fld[ne])
        for code, sgn in U_MIRROR.items():
            m = (~inner) & (bc[:, f] == code)
            for vp, vm in zip(vals_p, vals_m):
                vp[m] = sgn * vm[m]
        ubm, vbm, utm, vtm = vals_m
        ubp, vbp, utp, vtp = vals_p
        nx, ny = nxf[:, f][:, None], nyf[:, f][:, None]
        nUm, nUp = nx * ubm + ny * vbm, nx * ubp + ny * vbp
        lam = np.maximum(np.abs(nUm), np.abs(nUp))
        for c, (cm, cp) in enumerate(((utm, utp), (vtm, vtp))):
            flux = 0.5 * (nUm * cm + nUp * cp) + 0.5 * lam * (cm - cp)   # Alg. SSS, R27
            weak[c] += np.einsum("q,eqn,eq->en", wt, Lm, sJ[:, f][:, None] * flux)
    Minv = np.linalg.inv(ref.M)
    out = [(weak[c] @ Minv.T) / J[:, None] for c in range(2)]
    return out[0], out[1]


def face_flux_integrals(VX, VY, EToV, bc, ref, ub, vb, ut, vt):
    """Diagnostics for the pins: per component, (sum over boundary faces of the integral of n.F~*,
    1/2 sum over interior faces of Lambda [[c]]^2 integrated (each face once), 1/2 sum over boundary faces
    of (n.U_bar) c^2 integrated)."""
    N, Np = ref.N, ref.Np
    K = EToV.shape[0]
    geo = meshops.affine_geometry(VX, VY, EToV)
    nxf, nyf, sJ = meshops.face_geometry(VX, VY, EToV)
    EToE, _, _, _ = meshops.connectivity(VX, VY, EToV, bc, ref)
    tq, wt = line_rule(_npts(N))
    out = np.zeros((2, 3))
    e = np.arange(K)
    for f in range(3):
        a, b = EToV[e, f], EToV[e, (f + 1) % 3]
        px = VX[a][:, None] + (tq[None, :] + 1) / 2 * (VX[b] - VX[a])[:, None]
        py = VY[a][:, None] + (tq[None, :] + 1) / 2 * (VY[b] - VY[a])[:, None]
        r, s = _to_reference(geo["Jm"], VX[EToV[:, 0]], VY[EToV[:, 0]], px, py)
        Lm = ref.eval_basis(r.ravel(), s.ravel()).reshape(K, -1, Np)
        ubm, vbm, utm, vtm = (np.einsum("eqn,en->eq", Lm, fld) for fld in (ub, vb, ut, vt))
        nb = EToE[e, f]
        nx, ny = nxf[:, f][:, None], nyf[:, f][:, None]
        nUm = nx * ubm + ny * vbm
        for c, cm in enumerate((utm, vtm)):
            for code, sgn in U_MIRROR.items():
                m = (nb < 0) & (bc[:, f] == code)
                if not np.any(m):
                    continue
                nUp, cp = sgn * nUm[m], sgn * cm[m]
                lam = np.maximum(np.abs(nUm[m]), np.abs(nUp))
                flux = 0.5 * (nUm[m] * cm[m] + nUp * cp) + 0.5 * lam * (cm[m] - cp)
                out[c, 0] += np.sum(wt[None] * sJ[m, f][:, None] * flux)
                out[c, 2] += 0.5 * np.sum(wt[None] * sJ[m, f][:, None] * nUm[m] * cm[m] ** 2)
            inner = (nb >= 0) & (nb > e)  # each interior face once
            if np.any(inner):
                ne = nb[inner]
                rp, sp_ = _to_reference(geo["Jm"][ne], VX[EToV[ne, 0]], VY[EToV[ne, 0]], px[inner], py[inner])
                Lp = ref.eval_basis(rp.ravel(), sp_.ravel()).reshape(ne.size, -1, Np)
                ubp = np.einsum("eqn,en->eq", Lp, ub[ne])
                vbp = np.einsum("eqn,en->eq", Lp, vb[ne])
                cp = np.einsum("eqn,en->eq", Lp, (ut if c == 0 else vt)[ne])
                lam = np.maximum(np.abs(nUm[inner]), np.abs(nx[inner] * ubp + ny[inner] * vbp))
                out[c, 1] += 0.5 * np.sum(wt[None] * sJ[inner, f][:, None] * lam * (cm[inner] - cp) ** 2)
    return out
