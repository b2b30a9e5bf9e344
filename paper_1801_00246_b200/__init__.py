"""B200-native FP64 SIPDG Poisson operator and Jacobi-PCG (arXiv:1801.00246 hot path).

Thin Python layer over the C ABI of ``libipdg.so`` (include/ipdg.h).  Every
step of the operator and the solver runs in the library's CUDA kernels; this
module only marshals arguments.  PyTorch supplies device memory and streams
(tensors are passed by ``data_ptr()``; the stream defaults to
``torch.cuda.current_stream()``).  If the library is not built, calls raise.

    import torch
    from paper_1801_00246_b200 import Ipdg, meshgen
    mesh = meshgen.square(316, jitter=0.2, diag="random", order="morton", seed=2)
    op = Ipdg(N=4, mesh=mesh)
    u = torch.rand(op.K, op.Np, dtype=torch.float64, device="cuda")
    Au = op.ax(u)                                     # ipdg_ax
    x, stats = op.pcg_solve(b, tol=1e-8, maxit=5000)  # ipdg_pcg_solve (Jacobi by default)
    x, stats = op.pcg_solve(b, lam=1e3, precond=2)     # screened Poisson, block-Jacobi
    gx, gy = op.dg_grad(p); d = op.dg_div(ux, uy)       # DG gradient / divergence

Preconditioners (``precond``): 0 none, 1 point Jacobi diag(A), 2 block-Jacobi scaled inverse
mass (lambda > 0).
"""
import ctypes

import numpy as np

from . import _lib, meshgen  # noqa: F401
from ._lib import IpdgError, check, ipdg_stats, lib  # noqa: F401

__all__ = ["Ipdg", "IpdgError", "ipdg_stats", "lib", "meshgen"]


def _stream(stream):
    if stream is not None:
        return ctypes.c_void_p(int(stream))
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


class Ipdg:
    """One libipdg context (ipdg_create / ipdg_upload_mesh) bound to one CUDA device."""

    def __init__(self, N, mesh=None, device=0, tau_scale=1.0):
        self.N = int(N)
        self.Np = (self.N + 1) * (self.N + 2) // 2
        self.Nfp = self.N + 1
        self.device = int(device)
        self.ctx = ctypes.c_void_p()
        check(lib().ipdg_create(ctypes.byref(self.ctx), self.N, self.device))
        self.K = 0
        self._ws = None
        if mesh is not None:
            self.upload_mesh(mesh, tau_scale)

    def __del__(self):
        try:
            if self.ctx and self.ctx.value:
                lib().ipdg_destroy(self.ctx)
                self.ctx = ctypes.c_void_p()
        except Exception:
            pass

    @classmethod
    def from_rank_mesh(cls, N, rm, device=0, tau_scale=1.0, nccl_id=None):
        """Context for one partition (paper_1801_00246_b200.partition.RankMesh).

        With nccl_id (bytes of an ncclUniqueId shared by all ranks) the halo is exchanged with NCCL;
        without it the caller installs ghost rows with halo_set (single-process tests)."""
        op = cls(N, device=device)
        if nccl_id is not None:
            op.comm_init(nccl_id, rm.nparts, rm.rank)
        op.upload_mesh(rm.local_mesh(), tau_scale)
        if rm.H > 0 or (rm.bc == 3).any():
            ge = np.ascontiguousarray(rm.ghost_EToV, dtype=np.int32)
            rem = np.ascontiguousarray(rm.remote, dtype=np.int32)
            rf = np.ascontiguousarray(rm.remote_face, dtype=np.int8)
            nr = np.ascontiguousarray(rm.nbr_ranks, dtype=np.int32)
            so = np.ascontiguousarray(rm.send_off, dtype=np.int64)
            se = np.ascontiguousarray(rm.send_elems, dtype=np.int32)
            ro = np.ascontiguousarray(rm.recv_off, dtype=np.int64)
            check(lib().ipdg_upload_halo(op.ctx, rm.H, ge.ctypes.data, rem.ctypes.data, rf.ctypes.data, nr.size,
                                         nr.ctypes.data, so.ctypes.data, se.ctypes.data, ro.ctypes.data), op.ctx)
            op._ws = None  # the library dropped the workspace binding (its layout depends on K + H)
        op.rank_mesh = rm
        return op

    @classmethod
    def distributed(cls, N, mesh, part, rank, world, device=0, tau_scale=1.0):
        """One rank of a torch.distributed job: partition, NCCL bootstrap (id broadcast), upload."""
        import torch.distributed as dist
        from . import partition
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        rm = partition.split(mesh, part, world, ranks=[rank])[0]
        return cls.from_rank_mesh(N, rm, device=device, tau_scale=tau_scale, nccl_id=obj[0])

    def halo_info(self):
        S, H = ctypes.c_int64(), ctypes.c_int64()
        check(lib().ipdg_halo_info(self.ctx, ctypes.byref(S), ctypes.byref(H)), self.ctx)
        return S.value, H.value

    def halo_pack(self, u, stream=None):
        import torch
        S, _ = self.halo_info()
        out = torch.empty(max(S, 1), self.Np, dtype=torch.float64, device="cuda:%d" % self.device)
        check(lib().ipdg_halo_pack(self.ctx, _ptr(u), _ptr(out), _stream(stream)), self.ctx)
        return out[:S]

    def halo_set(self, ghosts, stream=None):
        check(lib().ipdg_halo_set(self.ctx, _ptr(ghosts.contiguous()), _stream(stream)), self.ctx)

    # ---- setup
    def comm_init(self, nccl_id_bytes, nranks, rank):
        buf = ctypes.create_string_buffer(bytes(nccl_id_bytes), len(nccl_id_bytes))
        check(lib().ipdg_comm_init(self.ctx, buf, int(nranks), int(rank)), self.ctx)

    def upload_mesh(self, mesh, tau_scale=1.0):
        VX = np.ascontiguousarray(mesh["VX"], dtype=np.float64)
        VY = np.ascontiguousarray(mesh["VY"], dtype=np.float64)
        EToV = np.ascontiguousarray(mesh["EToV"], dtype=np.int32)
        bc = np.ascontiguousarray(mesh["bc"], dtype=np.int8)
        K = EToV.shape[0]
        check(lib().ipdg_upload_mesh(self.ctx, K, VX.size, VX.ctypes.data, VY.ctypes.data, EToV.ctypes.data,
                                     bc.ctypes.data, float(tau_scale)), self.ctx)
        self.K = K
        self.rank_mesh = None
        self._ws = None

    def _workspace(self):
        if self._ws is None:
            import torch
            n = ctypes.c_int64()
            check(lib().ipdg_workspace_bytes(self.ctx, ctypes.byref(n)), self.ctx)
            self._ws = torch.empty(n.value, dtype=torch.uint8, device="cuda:%d" % self.device)
            check(lib().ipdg_set_workspace(self.ctx, _ptr(self._ws), n.value), self.ctx)
        return self._ws

    def _empty(self):
        import torch
        return torch.empty(self.K, self.Np, dtype=torch.float64, device="cuda:%d" % self.device)

    # ---- operator
    def ax(self, u, out=None, lam=0.0, stream=None):
        out = self._empty() if out is None else out
        check(lib().ipdg_ax(self.ctx, _ptr(u), _ptr(out), float(lam), _stream(stream)), self.ctx)
        return out

    def dg_grad(self, p, stream=None):
        """Nodal DG gradient with central fluxes, G p (Eq. INS_SD_4_1): returns (gx, gy)."""
        import torch
        gx, gy = torch.empty_like(p), torch.empty_like(p)
        check(lib().ipdg_dg_grad(self.ctx, _ptr(p), _ptr(gx), _ptr(gy), _stream(stream)), self.ctx)
        return gx, gy

    def dg_div(self, ux, uy, stream=None):
        """Nodal DG divergence with central fluxes, D u (Eq. INS_SD_4_2)."""
        import torch
        d = torch.empty_like(ux)
        check(lib().ipdg_dg_div(self.ctx, _ptr(ux), _ptr(uy), _ptr(d), _stream(stream)), self.ctx)
        return d

    def diag(self, lam=0.0, out=None, stream=None):
        out = self._empty() if out is None else out
        check(lib().ipdg_diag(self.ctx, _ptr(out), float(lam), _stream(stream)), self.ctx)
        return out

    def mass(self, u, out=None, stream=None):
        out = self._empty() if out is None else out
        check(lib().ipdg_mass(self.ctx, _ptr(u), _ptr(out), _stream(stream)), self.ctx)
        return out

    def nodes(self, stream=None):
        x, y = self._empty(), self._empty()
        check(lib().ipdg_nodes(self.ctx, _ptr(x), _ptr(y), _stream(stream)), self.ctx)
        return x, y

    # ---- solver
    def pcg_solve(self, b, x=None, lam=0.0, precond=1, tol=1e-8, maxit=10000, stream=None):
        self._workspace()
        if x is None:
            x = self._empty().zero_()
        st = ipdg_stats()
        rc = lib().ipdg_pcg_solve(self.ctx, _ptr(b), _ptr(x), float(lam), int(precond), float(tol), int(maxit),
                                  ctypes.byref(st), _stream(stream))
        check(rc, self.ctx, ok=(_lib.IPDG_OK, _lib.IPDG_NOT_CONVERGED))
        return x, dict(iterations=st.iterations, rel_residual=st.rel_residual, bnorm=st.bnorm, status=st.status, seconds=st.seconds)

    def pcg_begin(self, b, x, lam=0.0, precond=1, tol=1e-8, stream=None):
        self._workspace()
        check(lib().ipdg_pcg_begin(self.ctx, _ptr(b), _ptr(x), float(lam), int(precond), float(tol),
                                   _stream(stream)), self.ctx)

    def pcg_iterate(self, n, stream=None):
        check(lib().ipdg_pcg_iterate(self.ctx, int(n), _stream(stream)), self.ctx)

    def pcg_iterate_profiled(self, n, stream=None):
        """n iterations launched one by one with CUDA events around each pass: (ms_pass_a, ms_pass_b)."""
        ta, tb = ctypes.c_double(), ctypes.c_double()
        check(lib().ipdg_pcg_iterate_profiled(self.ctx, int(n), ctypes.byref(ta), ctypes.byref(tb), _stream(stream)),
              self.ctx)
        return ta.value, tb.value

    def pcg_end(self, stream=None):
        st = ipdg_stats()
        rc = lib().ipdg_pcg_end(self.ctx, ctypes.byref(st), _stream(stream))
        check(rc, self.ctx, ok=(_lib.IPDG_OK, _lib.IPDG_NOT_CONVERGED))
        return dict(iterations=st.iterations, rel_residual=st.rel_residual, bnorm=st.bnorm, status=st.status, seconds=st.seconds)

    def pcg_solve_host(self, b_host, x_host, lam=0.0, precond=1, tol=1e-8, maxit=10000, stream=None):
        """e2e path: host (pinned) numpy/torch CPU buffers in and out."""
        self._workspace()
        st = ipdg_stats()
        rc = lib().ipdg_pcg_solve_host(self.ctx, ctypes.c_void_p(b_host.data_ptr()), ctypes.c_void_p(x_host.data_ptr()),
                                       float(lam), int(precond), float(tol), int(maxit), ctypes.byref(st),
                                       _stream(stream))
        check(rc, self.ctx, ok=(_lib.IPDG_OK, _lib.IPDG_NOT_CONVERGED))
        return dict(iterations=st.iterations, rel_residual=st.rel_residual, bnorm=st.bnorm, status=st.status, seconds=st.seconds)

    def pmg_apply(self, r, out=None, lam=0.0, stream=None):
        """One p-multigrid V-cycle z = B r (the IPDG_PRECOND_PMG preconditioner)."""
        self._workspace()
        z = torch_empty_like(r) if out is None else out
        check(lib().ipdg_pmg_apply(self.ctx, _ptr(r), _ptr(z), float(lam), _stream(stream)), self.ctx)
        return z

    def advect(self, ub, vb, ut, vt, stream=None):
        """Subcycling advection operator (Nu, Nv) = N~(U_bar, U~) (ipdg_advect, NEXT-4)."""
        Nu, Nv = self._empty(), self._empty()
        check(lib().ipdg_advect(self.ctx, _ptr(ub), _ptr(vb), _ptr(ut), _ptr(vt), _ptr(Nu), _ptr(Nv),
                                _stream(stream)), self.ctx)
        return Nu, Nv

    def pmg_info(self):
        deg = (ctypes.c_int * 16)()
        lm = (ctypes.c_double * 16)()
        n = lib().ipdg_pmg_info(self.ctx, deg, lm, 16)
        check(min(n, 0), self.ctx)
        return [(deg[i], lm[i]) for i in range(n)]

    # ---- introspection
    def refop(self, name):
        n = {"r": self.Np, "s": self.Np, "Dr": self.Np ** 2, "Ds": self.Np ** 2, "M": self.Np ** 2,
             "M1D": self.Nfp ** 2, "LIFT": self.Np * 3 * self.Nfp, "Fmask": 3 * self.Nfp}[name]
        buf = np.zeros(n)
        got = lib().ipdg_get_refop(self.ctx, _lib.OPS[name], buf.ctypes.data, n)
        if got != n:
            check(got if got < 0 else _lib.IPDG_EINVAL, self.ctx)
        shape = {"Dr": (self.Np, self.Np), "Ds": (self.Np, self.Np), "M": (self.Np, self.Np),
                 "M1D": (self.Nfp, self.Nfp), "LIFT": (self.Np, 3 * self.Nfp), "Fmask": (3, self.Nfp)}.get(name)
        return buf.reshape(shape) if shape else buf

    def geofacs(self):
        buf = np.zeros(self.K * 5)
        check(lib().ipdg_get_geofacs(self.ctx, buf.ctypes.data, buf.size), self.ctx)
        return buf.reshape(self.K, 5)

    def connectivity(self):
        e = np.zeros(self.K * 3, dtype=np.int32)
        f = np.zeros(self.K * 3, dtype=np.int32)
        check(lib().ipdg_get_connectivity(self.ctx, e.ctypes.data, f.ctypes.data, e.size), self.ctx)
        return e.reshape(self.K, 3), f.reshape(self.K, 3)

    def info(self):
        out = (ctypes.c_int64 * 11)()
        check(lib().ipdg_info(self.ctx, out, 11), self.ctx)
        keys = ["N", "Np", "K", "nblocks", "E", "gmax", "smem_bytes", "grid", "kernel", "kernel_smem_bytes", "kernel_grid"]
        return dict(zip(keys, list(out)))

    def set_variant(self, variant):
        """0 auto, 1 fused (k_sipdg), 2 split (k_grad + k_flux), 4 pipelined fused (k_pipe),
        5 gather (k_gather, N <= 4)."""
        check(lib().ipdg_set_variant(self.ctx, int(variant)), self.ctx)

    def debug_grid_cap(self, cap):
        """Test hook (not in ipdg.h): cap every persistent grid at `cap` CTAs (0 = off), so a small mesh
        runs several element blocks per CTA through the kernels' prefetch pipelines."""
        fn = lib().ipdg_debug_grid_cap
        fn.restype = ctypes.c_int
        fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
        check(fn(self.ctx, int(cap)), self.ctx)

    def launch_count(self):
        return int(lib().ipdg_launch_count(self.ctx))


def loopback_pcg_solve(ops, bs, xs, lam=0.0, precond=1, tol=1e-8, maxit=10000, stream=None):
    """Distributed PCG over the partitions `ops` (Ipdg.from_rank_mesh contexts on one device, no NCCL)
    in lockstep: halo exchange by device copies, all-reduces by fixed-order sums (ipdg_loopback_pcg_solve).
    bs, xs: per-partition device tensors (xs hold x0, overwritten).  Returns per-partition stats."""
    P = len(ops)
    for op in ops:
        op._workspace()
    ctxs = (ctypes.c_void_p * P)(*[op.ctx.value for op in ops])
    bp = (ctypes.c_void_p * P)(*[b.data_ptr() for b in bs])
    xp = (ctypes.c_void_p * P)(*[x.data_ptr() for x in xs])
    st = (ipdg_stats * P)()
    rc = lib().ipdg_loopback_pcg_solve(ctxs, P, bp, xp, float(lam), int(precond), float(tol), int(maxit), st,
                                       _stream(stream))
    check(rc, ops[0].ctx, ok=(_lib.IPDG_OK, _lib.IPDG_NOT_CONVERGED))
    return [dict(iterations=s.iterations, rel_residual=s.rel_residual, bnorm=s.bnorm, status=s.status, seconds=s.seconds) for s in st]


def torch_empty_like(t):
    import torch
    return torch.empty_like(t)


def nccl_unique_id():
    n = lib().ipdg_nccl_id_bytes()
    buf = ctypes.create_string_buffer(n)
    check(lib().ipdg_nccl_get_unique_id(buf))
    return buf.raw


# expose the C names (same names as include/ipdg.h) for direct use
def __getattr__(name):
    if name.startswith("ipdg_") and name in _lib.SIGNATURES:
        return getattr(lib(), name)
    raise AttributeError(name)
