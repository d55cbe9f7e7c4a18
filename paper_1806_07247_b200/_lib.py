"""Thin ctypes binding of libtprod.so (include/tprod.h).  Argument marshalling only: every step
of the t-product runs in the library's CUDA kernels.  There is no CPU fallback -- if the shared
library is missing or the device is not a B200, calls raise."""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# TPROD_LIB overrides the in-tree library (A/B timing of two builds); default: the in-tree build
LIB_PATH = os.environ.get("TPROD_LIB") or os.path.join(_PKG, "libtprod.so")

TPROD_OK, TPROD_EINVAL, TPROD_EALIAS, TPROD_ENOMEM, TPROD_ECUDA, TPROD_ENCCL, \
    TPROD_EUNSUPPORTED, TPROD_ENOWORLD, TPROD_ESINGULAR = range(9)
TPROD_DTYPE_F32, TPROD_DTYPE_F64 = 0, 1
(TPROD_OPT_ENGINE, TPROD_OPT_GEMM_BN, TPROD_OPT_TIMING, TPROD_OPT_GEMM_CLUSTER, TPROD_OPT_TRANSFORM,
 TPROD_OPT_GRAPHS, TPROD_OPT_POISON, TPROD_OPT_SYNC_CHECKS, TPROD_OPT_OVERLAP,
 TPROD_OPT_FUSED_SCALES) = 1, 2, 3, 4, 5, 6, 7, 8, 9, 10
TPROD_STATUS_SINGULAR, TPROD_STATUS_NOCONVERGE = 1, 2

# name -> (restype, argtypes); the full list of symbols include/tprod.h declares
_i64, _vp, _int = C.c_int64, C.c_void_p, C.c_int
SIGNATURES = {
    "tprod_create": (_int, [_int, C.POINTER(_vp)]),
    "tprod_destroy": (_int, [_vp]),
    "tprod_f32": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp]),
    "tprod_f64": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp]),
    "tprod_f32_host": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp]),
    "tprod_f64_host": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp]),
    "tprod_workspace_bytes": (_int, [_i64, _i64, _i64, _i64, _int, C.POINTER(C.c_size_t)]),
    "tprod_strerror": (C.c_char_p, [_int]),
    "tprod_last_launch_count": (_int, [_vp, C.POINTER(_i64)]),
    "tprod_nccl_unique_id": (_int, [_vp]),
    "tprod_set_world": (_int, [_vp, _int, _int, _vp]),
    "tprod_bcast_f32": (_int, [_vp, _vp, _i64, _int, _vp]),
    "tprod_bcast_f64": (_int, [_vp, _vp, _i64, _int, _vp]),
    "tprod_dft_f32": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _int, _vp, _vp]),
    "tprod_idft_f32": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp]),
    "tprod_set_option": (_int, [_vp, _int, _i64]),
    "tprod_last_stage_ms": (_int, [_vp, C.POINTER(C.c_float)]),
    "tprod_status": (_int, [_vp, _vp, C.POINTER(_int)]),
    "tprod_prepare_a_f32": (_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "tprod_f32_prepared": (_int, [_vp, _vp, _i64, _vp, _vp]),
    "tprod_release_a": (_int, [_vp]),
    "tprod_tran_f32": (_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp]),
    "tprod_tran_f64": (_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp]),
    "tprod_teye_f32": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "tprod_teye_f64": (_int, [_vp, _i64, _i64, _vp, _vp]),
    "tprod_tinv_f32": (_int, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "tprod_tsvt_f32": (_int, [_vp, _vp, _i64, _i64, _i64, C.c_float, _vp, _vp]),
    "tprod_tsvd_values_f32": (_int, [_vp, _i64, _i64, _i64, C.c_float, _vp, _vp, _vp]),
    "tprod_tsvd_f32": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp]),
    "tprod_tsvd_full_f32": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libtprod.so (in-tree).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_1806_07247_b200.build` "
                              "(no CPU fallback exists)")
        l = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


class TprodError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {lib().tprod_strerror(status).decode()} (status {status})")


def check(status: int, what: str) -> None:
    if status != TPROD_OK:
        raise TprodError(status, what)


def strerror(status: int) -> str:
    return lib().tprod_strerror(status).decode()


def workspace_bytes(n1: int, n2: int, n3: int, n4: int, dtype: int = TPROD_DTYPE_F32) -> int:
    out = C.c_size_t()
    check(lib().tprod_workspace_bytes(n1, n2, n3, n4, dtype, C.byref(out)), "tprod_workspace_bytes")
    return out.value
