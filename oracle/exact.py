"""The SIPDG matrix in exact rational arithmetic for N <= 2 (oracle; test infrastructure only).

For N = 1 and N = 2 the Warp & Blend nodes are the equidistant lattice points
(the 1-D GLL points for N <= 2 are {-1, 1} and {-1, 0, 1}, so the warp
vanishes).  On meshes with dyadic vertex coordinates every
entry of the SIPDG matrix of oracle.assemble is then rational:
  * J, r_x, s_x, r_y, s_y are rational (Eq. operators2);
  * sJ n = (dy, -dx)/2 is rational although sJ = |edge|/2 need not be;
  * tau sJ = (N+1)(N+2)/2 sJ^2 max(1/J-, 1/J+) (Eq. Ch2.PenaltyParameter with
    1/h = |dE^f|/|E| = sJ/J) is rational.
The bilinear form (oracle.assemble docstring; Eq. ellipticOp1) is integrated
exactly: monomials over the bi-unit triangle in closed form, faces as
polynomials in the edge parameter t in [-1, 1].  Used to pin the float
oracle to ~1e-15 (tests/test_oracle_exact.py).
"""
from fractions import Fraction as Fr


# ---- polynomials in two variables: dict {(a, b): Fraction}
def padd(p, q, c=Fr(1)):
    out = dict(p)
    for k, v in q.items():
        out[k] = out.get(k, Fr(0)) + c * v
    return {k: v for k, v in out.items() if v != 0}


def pmul(p, q):
    out = {}
    for (a1, b1), v1 in p.items():
        for (a2, b2), v2 in q.items():
            k = (a1 + a2, b1 + b2)
            out[k] = out.get(k, Fr(0)) + v1 * v2
    return {k: v for k, v in out.items() if v != 0}


def pscale(p, c):
    return {k: v * c for k, v in p.items() if v * c != 0}


def pdiff(p, var):
    out = {}
    for (a, b), v in p.items():
        if var == 0 and a > 0:
            out[(a - 1, b)] = out.get((a - 1, b), Fr(0)) + a * v
        if var == 1 and b > 0:
            out[(a, b - 1)] = out.get((a, b - 1), Fr(0)) + b * v
    return out


def _line_moment(k):
    """int_{-1}^{1} t^k dt."""
    return Fr(2, k + 1) if k % 2 == 0 else Fr(0)


def tri_moment(a, b):
    """int over {r,s >= -1, r+s <= 0} of r^a s^b dr ds (closed form)."""
    return Fr((-1) ** (a + 1), a + 1) * (_line_moment(a + b + 1) - _line_moment(b))


def pint_tri(p):
    return sum((v * tri_moment(a, b) for (a, b), v in p.items()), Fr(0))


def compose_affine(p, r0, r1, s0, s1):
    """p(r0 + r1 t, s0 + s1 t) as a polynomial in t: dict {k: Fraction}."""
    out = {}
    for (a, b), v in p.items():
        poly = {0: v}
        for _ in range(a):
            poly = _mul1(poly, {0: r0, 1: r1})
        for _ in range(b):
            poly = _mul1(poly, {0: s0, 1: s1})
        for k, c in poly.items():
            out[k] = out.get(k, Fr(0)) + c
    return out


def _mul1(p, q):
    out = {}
    for k1, v1 in p.items():
        for k2, v2 in q.items():
            out[k1 + k2] = out.get(k1 + k2, Fr(0)) + v1 * v2
    return out


def pint_line(p):
    return sum((v * _line_moment(k) for k, v in p.items()), Fr(0))


# ---- reference nodes and Lagrange basis
def lattice_nodes(N):
    """Equidistant nodes for N <= 2, ordered row by row in s, r increasing (= Warp & Blend for N <= 2)."""
    if N not in (1, 2):
        raise ValueError("exact oracle supports N = 1, 2 only")
    pts = []
    for j in range(N + 1):
        for i in range(N + 1 - j):
            pts.append((Fr(-1) + Fr(2 * i, N), Fr(-1) + Fr(2 * j, N)))
    return pts


def _solve(Am, B):
    """Gauss-Jordan on Fractions: returns X with Am X = B (lists of lists)."""
    n = len(Am)
    M = [list(Am[i]) + list(B[i]) for i in range(n)]
    for c in range(n):
        piv = next(i for i in range(c, n) if M[i][c] != 0)
        M[c], M[piv] = M[piv], M[c]
        pv = M[c][c]
        M[c] = [x / pv for x in M[c]]
        for i in range(n):
            if i != c and M[i][c] != 0:
                f = M[i][c]
                M[i] = [x - f * y for x, y in zip(M[i], M[c])]
    return [row[n:] for row in M]


def lagrange_basis(N):
    """Exact Lagrange polynomials l_i(r,s) on the lattice nodes (monomial coefficients)."""
    pts = lattice_nodes(N)
    mons = [(a, b) for a in range(N + 1) for b in range(N + 1 - a)]
    V = [[r ** a * s ** b for (a, b) in mons] for (r, s) in pts]
    n = len(pts)
    I = [[Fr(int(i == j)) for j in range(n)] for i in range(n)]
    C = _solve(V, I)  # V C = I: column i holds coefficients of l_i
    return [{mons[k]: C[k][i] for k in range(n) if C[k][i] != 0} for i in range(n)]


def assemble_exact(VX, VY, EToV, bc, N, lam=Fr(0)):
    """Dense exact SIPDG matrix (list of lists of Fraction) of size K*Np."""
    basis = lagrange_basis(N)
    Np = len(basis)
    K = len(EToV)
    X = [Fr(float(x)) for x in VX]
    Y = [Fr(float(y)) for y in VY]
    dr = [pdiff(p, 0) for p in basis]
    ds = [pdiff(p, 1) for p in basis]
    geo = []
    for e in range(K):
        v = [int(t) for t in EToV[e]]
        xr, xs = (X[v[1]] - X[v[0]]) / 2, (X[v[2]] - X[v[0]]) / 2
        yr, ys = (Y[v[1]] - Y[v[0]]) / 2, (Y[v[2]] - Y[v[0]]) / 2
        J = xr * ys - xs * yr
        geo.append(dict(v=v, xr=xr, xs=xs, yr=yr, ys=ys, J=J, rx=ys / J, ry=-xs / J, sx=-yr / J, sy=xr / J))
    n = K * Np
    A = [[Fr(0)] * n for _ in range(n)]

    def grad_phys(g):
        gx = [padd(pscale(dr[i], g["rx"]), pscale(ds[i], g["sx"])) for i in range(Np)]
        gy = [padd(pscale(dr[i], g["ry"]), pscale(ds[i], g["sy"])) for i in range(Np)]
        return gx, gy

    grads = [grad_phys(g) for g in geo]
    # volume
    for e in range(K):
        gx, gy = grads[e]
        J = geo[e]["J"]
        for i in range(Np):
            for j in range(Np):
                val = pint_tri(padd(pmul(gx[i], gx[j]), pmul(gy[i], gy[j]))) * J
                if lam:
                    val += lam * J * pint_tri(pmul(basis[i], basis[j]))
                A[e * Np + i][e * Np + j] += val
    # faces
    edges = {}
    for e in range(K):
        for f in range(3):
            a, b = geo[e]["v"][f], geo[e]["v"][(f + 1) % 3]
            edges.setdefault(tuple(sorted((a, b))), []).append((e, f))
    c = Fr((N + 1) * (N + 2), 2)

    def trace(e, a, b):
        """Basis values and (sJ n).grad (n outward of the element owning a->b) as polys in t."""
        g = geo[e]
        x1, y1 = X[g["v"][0]], Y[g["v"][0]]
        # x(t) = X[a] + (t+1)/2 (X[b]-X[a]) = (X[a]+X[b])/2 + t (X[b]-X[a])/2
        px0, px1 = (X[a] + X[b]) / 2 - x1, (X[b] - X[a]) / 2
        py0, py1 = (Y[a] + Y[b]) / 2 - y1, (Y[b] - Y[a]) / 2
        # (r+1, s+1) = inv(Jm) (x - x1), inv(Jm) = [[rx, ry],[sx, sy]]
        r0 = g["rx"] * px0 + g["ry"] * py0 - 1
        r1 = g["rx"] * px1 + g["ry"] * py1
        s0 = g["sx"] * px0 + g["sy"] * py0 - 1
        s1 = g["sx"] * px1 + g["sy"] * py1
        gx, gy = grads[e]
        return r0, r1, s0, s1, gx, gy

    for key, lst in edges.items():
        e, f = lst[0]
        g = geo[e]
        a, b = g["v"][f], g["v"][(f + 1) % 3]
        dx, dy = X[b] - X[a], Y[b] - Y[a]
        snx, sny = dy / 2, -dx / 2  # sJ * n, n outward of e
        sJ2 = (dx * dx + dy * dy) / 4
        r0, r1, s0, s1, gx, gy = trace(e, a, b)
        vm = [compose_affine(basis[i], r0, r1, s0, s1) for i in range(Np)]
        dm = [compose_affine(padd(pscale(gx[i], snx), pscale(gy[i], sny)), r0, r1, s0, s1) for i in range(Np)]
        # ds = sJ dt; (d_n phi, psi)_f = int (sJ n . grad phi) psi dt; tau (phi,psi)_f = tau sJ int phi psi dt
        if len(lst) == 1:
            code = int(bc[e][f])
            if code == 2:
                continue
            tsJ = c * sJ2 / g["J"]
            for i in range(Np):
                for j in range(Np):
                    val = (-pint_line(_mul1(dm[j], vm[i])) - pint_line(_mul1(dm[i], vm[j]))
                           + 2 * tsJ * pint_line(_mul1(vm[i], vm[j])))
                    A[e * Np + i][e * Np + j] += val
            continue
        (e2, f2) = lst[1]
        tsJ = c * sJ2 * max(1 / g["J"], 1 / geo[e2]["J"])
        r0p, r1p, s0p, s1p, gxp, gyp = trace(e2, a, b)
        vp = [compose_affine(basis[i], r0p, r1p, s0p, s1p) for i in range(Np)]
        dp = [compose_affine(padd(pscale(gxp[i], snx), pscale(gyp[i], sny)), r0p, r1p, s0p, s1p) for i in range(Np)]
        # stacked dofs: <phi> = phi- - phi+, {d_n phi} = d_n phi / 2 (n of e)
        dofs = [e * Np + i for i in range(Np)] + [e2 * Np + i for i in range(Np)]
        jmp = vm + [{k: -v for k, v in p.items()} for p in vp]
        avg = [{k: v / 2 for k, v in p.items()} for p in dm + dp]
        for i in range(2 * Np):
            for j in range(2 * Np):
                val = (-pint_line(_mul1(avg[j], jmp[i])) - pint_line(_mul1(avg[i], jmp[j]))
                       + tsJ * pint_line(_mul1(jmp[i], jmp[j])))
                A[dofs[i]][dofs[j]] += val
    return A
