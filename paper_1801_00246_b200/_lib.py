"""ctypes binding of libipdg.so (include/ipdg.h).  Argument marshalling only.

The shared library is built in-tree (``paper_1801_00246_b200/libipdg.so``) by
``paper_1801_00246_b200.build.build_library`` / ``__graft_entry__.build()``.
There is no fallback: if the library is missing or fails to load, every entry
point raises ``RuntimeError``.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IPDG_LIB") or os.path.join(HERE, "libipdg.so")  # IPDG_LIB: A/B timing of library builds
HEADER = os.path.join(os.path.dirname(HERE), "include", "ipdg.h")

IPDG_OK = 0
IPDG_NOT_CONVERGED = 1
IPDG_EINVAL = -1
IPDG_EDEGREE = -2
IPDG_EMESH = -3
IPDG_EBREAKDOWN = -4
IPDG_ESINGULAR = -5
IPDG_ECUDA = -6
IPDG_ENCCL = -7
IPDG_ESTATE = -8
OPS = dict(r=0, s=1, Dr=2, Ds=3, M=4, M1D=5, LIFT=6, Fmask=7)


class ipdg_stats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("rel_residual", ctypes.c_double), ("bnorm", ctypes.c_double),
                ("status", ctypes.c_int32), ("reserved", ctypes.c_int32), ("seconds", ctypes.c_double)]


_c = ctypes
_vp, _i64, _i32, _d, _int = _c.c_void_p, _c.c_int64, _c.c_int32, _c.c_double, _c.c_int
SIGNATURES = {
    "ipdg_create": (_int, [_c.POINTER(_vp), _int, _int]),
    "ipdg_destroy": (_int, [_vp]),
    "ipdg_upload_mesh": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _d]),
    "ipdg_ax": (_int, [_vp, _vp, _vp, _d, _vp]),
    "ipdg_diag": (_int, [_vp, _vp, _d, _vp]),
    "ipdg_mass": (_int, [_vp, _vp, _vp, _vp]),
    "ipdg_dg_grad": (_int, [_vp, _vp, _vp, _vp, _vp]),
    "ipdg_dg_div": (_int, [_vp, _vp, _vp, _vp, _vp]),
    "ipdg_nodes": (_int, [_vp, _vp, _vp, _vp]),
    "ipdg_workspace_bytes": (_int, [_vp, _c.POINTER(_i64)]),
    "ipdg_set_workspace": (_int, [_vp, _vp, _i64]),
    "ipdg_pcg_solve": (_int, [_vp, _vp, _vp, _d, _int, _d, _i64, _c.POINTER(ipdg_stats), _vp]),
    "ipdg_pcg_begin": (_int, [_vp, _vp, _vp, _d, _int, _d, _vp]),
    "ipdg_pcg_iterate": (_int, [_vp, _i64, _vp]),
    "ipdg_pcg_end": (_int, [_vp, _c.POINTER(ipdg_stats), _vp]),
    "ipdg_pcg_iterate_profiled": (_int, [_vp, _i64, _c.POINTER(_d), _c.POINTER(_d), _vp]),
    "ipdg_pcg_solve_host": (_int, [_vp, _vp, _vp, _d, _int, _d, _i64, _c.POINTER(ipdg_stats), _vp]),
    "ipdg_comm_init": (_int, [_vp, _vp, _int, _int]),
    "ipdg_pmg_apply": (_int, [_vp, _vp, _vp, _d, _vp]),
    "ipdg_advect": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ipdg_pmg_info": (_int, [_vp, _vp, _vp, _int]),
    "ipdg_loopback_pcg_solve": (_int, [_vp, _int, _vp, _vp, _d, _int, _d, _i64, _c.POINTER(ipdg_stats), _vp]),
    "ipdg_upload_halo": (_int, [_vp, _i64, _vp, _vp, _vp, _int, _vp, _vp, _vp, _vp]),
    "ipdg_halo_info": (_int, [_vp, _c.POINTER(_i64), _c.POINTER(_i64)]),
    "ipdg_halo_pack": (_int, [_vp, _vp, _vp, _vp]),
    "ipdg_halo_set": (_int, [_vp, _vp, _vp]),
    "ipdg_nccl_id_bytes": (_int, []),
    "ipdg_nccl_get_unique_id": (_int, [_vp]),
    "ipdg_get_refop": (_int, [_vp, _int, _vp, _i64]),
    "ipdg_refop_host": (_int, [_int, _int, _vp, _i64]),
    "ipdg_get_geofacs": (_int, [_vp, _vp, _i64]),
    "ipdg_get_connectivity": (_int, [_vp, _vp, _vp, _i64]),
    "ipdg_info": (_int, [_vp, _c.POINTER(_i64), _int]),
    "ipdg_launch_count": (_i64, [_vp]),
    "ipdg_set_variant": (_int, [_vp, _int]),
    "ipdg_strerror": (_c.c_char_p, [_int]),
    "ipdg_last_error": (_int, [_vp, _c.c_char_p, _int]),
}

_LIB = None


def lib():
    """Load libipdg.so once (RTLD_GLOBAL so NCCL symbols resolve once per process)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libipdg.so not built (%s); run __graft_entry__.build()" % LIB_PATH)
        import torch  # noqa: F401  -- torch's CUDA/NCCL libraries first; libipdg links the same libnccl.so.2
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


class IpdgError(RuntimeError):
    def __init__(self, code, detail):
        self.code = code
        super().__init__("ipdg error %d (%s): %s" % (code, lib().ipdg_strerror(code).decode(), detail))


def check(code, ctx=None, ok=(IPDG_OK,)):
    if code in ok:
        return code
    detail = ""
    if ctx is not None and ctx.value:
        buf = ctypes.create_string_buffer(512)
        lib().ipdg_last_error(ctx, buf, 512)
        detail = buf.value.decode(errors="replace")
    raise IpdgError(code, detail)
