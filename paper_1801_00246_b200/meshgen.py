"""Seeded synthetic inputs shared by the CUDA path and the oracle.

This module holds NONE of the method's arithmetic (no nodes, operators,
geometric factors, penalties or fluxes).  It produces only what a user would
hand to the solver: vertex coordinates, counter-clockwise triangles, a
boundary code per element face, an element ordering and a partition, plus
seeded random nodal fields.  Both sides of every parity test receive the same
arrays from here.

Mesh dict: VX, VY (Nv,) float64; EToV (K,3) int32 CCW; bc (K,3) int8 with
face f = edge {EToV[e,f], EToV[e,(f+1)%3]} and codes
  0 interior, 1 Dirichlet, 2 Neumann.
Workload shapes (BASELINE.json configs):
  C1 square(4, 4)                       32 triangles, "/" diagonals, no jitter
  C2 square(316, 316, jitter, random)   199,712 triangles, Morton order
  C3 square(707, 707, ...)              999,698 triangles
  C4 cylinder(...)                      graded channel [-16,25]x[-22,22] minus [-0.5,0.5]^2
  C5 tiles(1414, px, py)                one 1414x1414-cell tile per rank
"""
import numpy as np

INTERIOR, DIRICHLET, NEUMANN = 0, 1, 2


def _edge_codes(EToV, VX, VY, tag):
    """Boundary code per element face: faces seen once get tag(xm, ym) at the edge midpoint."""
    K = EToV.shape[0]
    a = EToV[:, [0, 1, 2]]
    b = EToV[:, [1, 2, 0]]
    lo = np.minimum(a, b).astype(np.int64)
    hi = np.maximum(a, b).astype(np.int64)
    key = lo * (int(EToV.max()) + 1) + hi
    flat = key.ravel()
    uniq, inv, cnt = np.unique(flat, return_inverse=True, return_counts=True)
    once = (cnt[inv] == 1).reshape(K, 3)
    bc = np.zeros((K, 3), dtype=np.int8)
    if np.any(once):
        xm = 0.5 * (VX[a] + VX[b])
        ym = 0.5 * (VY[a] + VY[b])
        codes = tag(xm[once], ym[once])
        bc[once] = np.asarray(codes, dtype=np.int8)
    if np.any(cnt > 2):
        raise ValueError("non-manifold edge in generated mesh")
    return bc


def _signed_area2(VX, VY, EToV):
    x = VX[EToV]
    y = VY[EToV]
    return (x[:, 1] - x[:, 0]) * (y[:, 2] - y[:, 0]) - (x[:, 2] - x[:, 0]) * (y[:, 1] - y[:, 0])


def morton_order(VX, VY, EToV):
    """Permutation sorting elements by the Z-order key of their vertex-mean point."""
    cx = VX[EToV].mean(axis=1)
    cy = VY[EToV].mean(axis=1)
    span = max(cx.max() - cx.min(), cy.max() - cy.min(), 1e-300)
    qx = np.clip(((cx - cx.min()) / span * 65535).astype(np.uint64), 0, 65535)
    qy = np.clip(((cy - cy.min()) / span * 65535).astype(np.uint64), 0, 65535)

    def spread(v):
        v = v & np.uint64(0xFFFF)
        v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF)
        v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F)
        v = (v | (v << np.uint64(2))) & np.uint64(0x33333333)
        v = (v | (v << np.uint64(1))) & np.uint64(0x55555555)
        return v

    key = spread(qx) | (spread(qy) << np.uint64(1))
    return np.argsort(key, kind="stable")


def _finish(VX, VY, EToV, tag, order, seed):
    if order == "morton":
        perm = morton_order(VX, VY, EToV)
        EToV = EToV[perm]
    elif order == "random":
        perm = np.random.default_rng(seed + 7).permutation(EToV.shape[0])
        EToV = EToV[perm]
    elif order != "natural":
        raise ValueError("order must be natural|morton|random")
    EToV = np.ascontiguousarray(EToV, dtype=np.int32)
    bc = _edge_codes(EToV, VX, VY, tag)
    return dict(VX=np.ascontiguousarray(VX, dtype=np.float64), VY=np.ascontiguousarray(VY, dtype=np.float64),
                EToV=EToV, bc=bc)


def _grid_triangles(xs, ys, diag, rng, keep=None):
    """Triangles of the tensor grid xs x ys; diag '/', '\\' or 'random'; keep(i,j) masks cells."""
    nx, ny = len(xs) - 1, len(ys) - 1
    X, Y = np.meshgrid(xs, ys, indexing="xy")  # (ny+1, nx+1)
    VX, VY = X.ravel().copy(), Y.ravel().copy()
    I, Jj = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    I, Jj = I.ravel(), Jj.ravel()
    if keep is not None:
        m = keep(I, Jj)
        I, Jj = I[m], Jj[m]
    v00 = Jj * (nx + 1) + I
    v10 = v00 + 1
    v01 = v00 + (nx + 1)
    v11 = v01 + 1
    if diag == "/":
        slash = np.ones(I.size, dtype=bool)
    elif diag == "\\":
        slash = np.zeros(I.size, dtype=bool)
    else:
        slash = rng.random(I.size) < 0.5
    t1 = np.where(slash[:, None], np.stack([v00, v10, v11], 1), np.stack([v00, v10, v01], 1))
    t2 = np.where(slash[:, None], np.stack([v00, v11, v01], 1), np.stack([v10, v11, v01], 1))
    EToV = np.empty((2 * I.size, 3), dtype=np.int64)
    EToV[0::2] = t1
    EToV[1::2] = t2
    used = np.unique(EToV)
    remap = -np.ones(VX.size, dtype=np.int64)
    remap[used] = np.arange(used.size)
    return VX[used], VY[used], remap[EToV]


def _jitter(VX, VY, EToV, h, jitter, rng, movable):
    for attempt in range(20):
        dx = (rng.random(VX.size) * 2 - 1) * jitter * h
        dy = (rng.random(VY.size) * 2 - 1) * jitter * h
        nx_, ny_ = VX + np.where(movable, dx, 0), VY + np.where(movable, dy, 0)
        if np.all(_signed_area2(nx_, ny_, EToV) > 0):
            return nx_, ny_
        jitter *= 0.7
    raise RuntimeError("could not jitter the mesh without inverting an element")


def square(nx, ny=None, x0=0.0, x1=1.0, y0=0.0, y1=1.0, jitter=0.0, diag="/", order="natural",
           seed=0, bc_code=DIRICHLET, tag=None):
    """Triangulated rectangle with 2*nx*ny triangles.

    jitter: interior vertices moved uniformly by up to jitter*h per coordinate (C2/C3: 0.2).
    diag: '/', '\\' or 'random' (C2/C3: random).  order: natural | morton | random.
    tag(xm, ym) -> code overrides the uniform boundary code bc_code.
    """
    ny = nx if ny is None else ny
    rng = np.random.default_rng(seed)
    xs = np.linspace(x0, x1, nx + 1)
    ys = np.linspace(y0, y1, ny + 1)
    VX, VY, EToV = _grid_triangles(xs, ys, diag, rng)
    if jitter > 0:
        h = min((x1 - x0) / nx, (y1 - y0) / ny)
        eps = 1e-12 * max(x1 - x0, y1 - y0)
        movable = (VX > x0 + eps) & (VX < x1 - eps) & (VY > y0 + eps) & (VY < y1 - eps)
        VX, VY = _jitter(VX, VY, EToV, h, jitter, rng, movable)
    tag = tag or (lambda xm, ym: np.full(xm.shape, bc_code, dtype=np.int8))
    return _finish(VX, VY, EToV, tag, order, seed)


def graded_axis(a, b, c0, c1, h0, ratio):
    """Coordinates from a to b that include [c0, c1] with spacing h0 inside, growing by `ratio` outside."""
    inner = np.linspace(c0, c1, int(round((c1 - c0) / h0)) + 1)

    def grow(length):
        pts, h, x = [0.0], h0, 0.0
        while x + h < length:
            x += h
            pts.append(x)
            h *= ratio
        if length - pts[-1] < 0.5 * h and len(pts) > 1:
            pts[-1] = length
        else:
            pts.append(length)
        return np.array(pts)

    left = c0 - grow(c0 - a)[::-1]
    right = c1 + grow(b - c1)
    return np.concatenate([left[:-1], inner, right[1:]])


def cylinder(h0=0.01, ratio=1.006, jitter=0.15, order="morton", seed=4):
    """Channel [-16,25]x[-22,22] minus the square cylinder [-0.5,0.5]^2, graded mesh.

    Pressure-Poisson boundary codes (SURVEY reading #9): outflow x = 25 Dirichlet;
    inflow x = -16, walls y = +-22 and the cylinder Neumann.  The defaults give about
    1.0 M cells = 2.0 M triangles (BASELINE config C4).
    """
    rng = np.random.default_rng(seed)
    xs = graded_axis(-16.0, 25.0, -0.5, 0.5, h0, ratio)
    ys = graded_axis(-22.0, 22.0, -0.5, 0.5, h0, ratio)
    cx = 0.5 * (xs[:-1] + xs[1:])
    cy = 0.5 * (ys[:-1] + ys[1:])

    def keep(i, j):
        return ~((np.abs(cx[i]) < 0.5) & (np.abs(cy[j]) < 0.5))

    VX, VY, EToV = _grid_triangles(xs, ys, "random", rng, keep)
    if jitter > 0:
        # move only vertices off every boundary; jitter scaled by the local spacing
        eps = 1e-9
        on_bnd = ((np.abs(VX + 16) < eps) | (np.abs(VX - 25) < eps) | (np.abs(VY + 22) < eps)
                  | (np.abs(VY - 22) < eps) | ((np.abs(VX) <= 0.5 + eps) & (np.abs(VY) <= 0.5 + eps)))
        ix = np.clip(np.searchsorted(xs, VX), 1, len(xs) - 1)
        iy = np.clip(np.searchsorted(ys, VY), 1, len(ys) - 1)
        hloc = np.minimum(np.diff(xs)[np.minimum(ix - 1, len(xs) - 2)], np.diff(ys)[np.minimum(iy - 1, len(ys) - 2)])
        hx = np.minimum(hloc, np.diff(xs)[np.minimum(ix, len(xs) - 2)])
        hy = np.minimum(hloc, np.diff(ys)[np.minimum(iy, len(ys) - 2)])
        for attempt in range(20):
            dx = (rng.random(VX.size) * 2 - 1) * jitter * hx
            dy = (rng.random(VY.size) * 2 - 1) * jitter * hy
            nx_, ny_ = VX + np.where(on_bnd, 0, dx), VY + np.where(on_bnd, 0, dy)
            if np.all(_signed_area2(nx_, ny_, EToV) > 0):
                VX, VY = nx_, ny_
                break
            jitter *= 0.7

    def tag(xm, ym):
        return np.where(np.abs(xm - 25.0) < 1e-9, DIRICHLET, NEUMANN).astype(np.int8)

    return _finish(VX, VY, EToV, tag, order, seed)


def tiles(n, px, py, jitter=0.2, seed=5):
    """px*py unit tiles of n x n cells each over [0,px]x[0,py] (C5 weak scaling), all-Dirichlet.

    Elements are grouped tile by tile (Morton order inside each tile); returns the mesh and
    `part` (K,) = the tile index (rank) of each element.
    """
    meshes = []
    for ty in range(py):
        for tx in range(px):
            m = square(n, n, tx, tx + 1.0, ty, ty + 1.0, jitter=0.0, diag="random", order="morton",
                       seed=seed + 101 * (ty * px + tx))
            meshes.append(m)
    # merge coincident vertices along tile seams by exact coordinate keys
    VXa = np.concatenate([m["VX"] for m in meshes])
    VYa = np.concatenate([m["VY"] for m in meshes])
    offs = np.cumsum([0] + [m["VX"].size for m in meshes])
    keys = np.round(VXa * n).astype(np.int64) * (py * n + 1 + 7) + np.round(VYa * n).astype(np.int64)
    uniq, inv = np.unique(keys, return_inverse=True)
    VX = np.zeros(uniq.size)
    VY = np.zeros(uniq.size)
    VX[inv] = VXa
    VY[inv] = VYa
    EToV = np.concatenate([inv[m["EToV"] + offs[i]] for i, m in enumerate(meshes)])
    part = np.concatenate([np.full(m["EToV"].shape[0], i, dtype=np.int32) for i, m in enumerate(meshes)])
    rng = np.random.default_rng(seed)
    if jitter > 0:
        eps = 1e-12
        movable = (VX > eps) & (VX < px - eps) & (VY > eps) & (VY < py - eps)
        VX, VY = _jitter(VX, VY, EToV, 1.0 / n, jitter, rng, movable)
    mesh = _finish(VX, VY, EToV, lambda xm, ym: np.full(xm.shape, DIRICHLET, dtype=np.int8), "natural", seed)
    return mesh, part


def rcb_partition(VX, VY, EToV, nparts):
    """Recursive coordinate bisection of elements by vertex-mean point; balanced counts."""
    cx = VX[EToV].mean(axis=1)
    cy = VY[EToV].mean(axis=1)
    part = np.zeros(EToV.shape[0], dtype=np.int32)

    def rec(idx, p0, np_):
        if np_ == 1:
            part[idx] = p0
            return
        nl = np_ // 2
        x, y = cx[idx], cy[idx]
        key = x if (x.max() - x.min()) >= (y.max() - y.min()) else y
        o = np.argsort(key, kind="stable")
        cut = (idx.size * nl) // np_
        rec(idx[o[:cut]], p0, nl)
        rec(idx[o[cut:]], p0 + nl, np_ - nl)

    rec(np.arange(EToV.shape[0]), 0, nparts)
    return part


def uniform_field(K, Np, seed):
    """u ~ U(-1, 1), shape (K, Np), float64 (operator inputs, seed 100+N)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(K, Np))


def sin_sin(x, y):
    """Manufactured solution of config C1 (BASELINE.json configs[0]): u = sin(pi x) sin(pi y)."""
    return np.sin(np.pi * x) * np.sin(np.pi * y)


def sin_sin_forcing(x, y):
    """f = -Laplace(u) = 2 pi^2 sin(pi x) sin(pi y) for u = sin_sin."""
    return 2 * np.pi ** 2 * np.sin(np.pi * x) * np.sin(np.pi * y)
