"""ctypes binding of the C ABI declared in include/strom_b200.h.

The product path has no CPU fallback: if the sm_100a library is missing this
module raises at import time, and every call requires CUDA tensors.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libstrom_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a library first "
        "(python paper_1910_01260_b200/_build.py or __graft_entry__.build())")

lib = C.CDLL(LIB_PATH)

i32, i64, dbl, vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p
P_I32 = C.POINTER(C.c_int32)


class IsvdInfo(C.Structure):
    _fields_ = [
        ("n", i64), ("k", i64), ("rank", i32), ("ncols_u", i32),
        ("n_rejected", i32), ("n_dependent", i32), ("n_truncated", i32), ("n_restarts", i32),
        ("flags", i32), ("status", i32),
        ("last_p", dbl), ("last_drift", dbl), ("last_xnorm", dbl),
        ("tol_svd", dbl), ("tol_sv", dbl), ("r_max", i64), ("cap_mode", i32), ("pad", i32),
        ("last_p_sq", dbl),
    ]


_PROTOS = {
    "strom_last_error": (C.c_char_p, []),
    "strom_abi_version": (C.c_int, []),
    "strom_device_synchronize": (C.c_int, []),
    "strom_profile_enable": (None, [i32]),
    "strom_trim_cache": (None, []),
    "strom_profile_reset": (C.c_int, []),
    "strom_profile_read": (C.c_int, [i32, C.POINTER(i64), C.POINTER(dbl), C.POINTER(dbl)]),
    "strom_profile_durations": (C.c_int, [i32, i32, C.POINTER(C.c_float), C.POINTER(i32)]),
    "strom_fp64_probe": (C.c_int, [i32, i32, vp, C.POINTER(dbl)]),
    "strom_isvd_init": (C.c_int, [i64, vp, i64, dbl, dbl, i64, i32, vp, C.POINTER(vp)]),
    "strom_isvd_update": (C.c_int, [vp, vp, vp, C.POINTER(vp)]),
    "strom_isvd_ingest": (C.c_int, [vp, vp, i64, i64, i32, vp, C.POINTER(vp)]),
    "strom_isvd_query": (C.c_int, [vp, vp, C.POINTER(IsvdInfo)]),
    "strom_isvd_export": (C.c_int, [vp, vp, vp, vp, vp]),
    "strom_isvd_load": (C.c_int, [i64, i64, i64, vp, vp, vp, dbl, dbl, i64, i32, P_I32, vp, C.POINTER(vp)]),
    "strom_isvd_load_factored": (C.c_int, [i64, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, vp,
                                           dbl, dbl, i64, i32, P_I32, vp, C.POINTER(vp)]),
    "strom_isvd_factors": (C.c_int, [vp, vp, vp, vp, vp]),
    "strom_debug_tprobe": (None, [vp]),
    "strom_debug_lu_probe": (None, [vp]),
    "strom_debug_trace": (None, [vp, i64]),
    "strom_debug_pass_bw": (C.c_int, [i64, i32, i32, i32, C.POINTER(dbl)]),
    "strom_isvd_free": (None, [vp]),
    # row-shard groups (csrc/shard.cuh)
    "strom_shard_mailbox_create": (C.c_int, [i32, C.POINTER(vp), vp]),
    "strom_shard_connect": (C.c_int, [vp, i32, i64, vp]),
    "strom_shard_create_local": (C.c_int, [i32, i64, C.POINTER(vp)]),
    "strom_shard_make_current": (None, [vp]),
    "strom_shard_status": (C.c_int, [vp, C.POINTER(i64), C.POINTER(i32)]),
    "strom_shard_free": (None, [vp]),
    # temporal bases (basis.py:275-302)
    "strom_temporal_bases": (C.c_int, [vp, i64, i64, i64, i64, i64, i64, vp, vp, vp, vp]),
    # spatial ROM (spatial.py:45-67)
    "strom_dense_lu": (C.c_int, [i64, vp, vp, vp]),
    "strom_dense_lu_solve": (C.c_int, [i64, vp, vp, vp, i64, vp]),
    "strom_st_apply_inverse": (C.c_int, [i64, i32, vp, vp, vp, vp, i64, dbl, i32, vp, P_I32, vp]),
    "strom_fom_march": (C.c_int, [i64, i32, vp, vp, vp, i64, vp, vp, vp, i64, dbl, i32, vp, P_I32, vp]),
    "strom_fom_march_tridiag": (C.c_int, [i64, vp, vp, vp, i32, vp, i64, vp, vp, vp, vp, i64, vp, vp]),
    "strom_gen_lowrank_batch": (C.c_int, [i64, i32, i32, vp, vp, C.c_uint64, i64, dbl, vp, i64, vp]),
    "strom_csr_to_ell": (C.c_int, [i64, vp, vp, vp, i32, i32, vp, vp, C.POINTER(i64), vp]),
    "strom_csr_spmm": (C.c_int, [i64, vp, vp, vp, i32, vp, i64, i64, vp, i64, vp]),
    "strom_spatial_reduce_ell": (C.c_int, [i64, i32, vp, vp, i64, vp, i64, i64, vp, i64, i64, vp, vp, vp]),
    "strom_spatial_reduce_csr": (C.c_int, [i64, vp, vp, vp, i32, vp, i64, i64, i64, vp, i64, i64, vp, vp,
                                           vp]),
    # space-time assembly (spacetime.py:43-115)
    "strom_st_assemble": (C.c_int, [vp, vp, vp, i64, i64, i64, vp, i64, vp, i32, vp, vp, vp, vp, vp]),
    "strom_st_reconstruct": (C.c_int, [i64, i64, i64, i64, vp, i64, vp, vp, vp, i64, vp]),
    # dense LU solve (linalg.py:75-99)
    "strom_dense_solve": (C.c_int, [i64, vp, vp, i64, vp, vp, vp]),
    # small SVD / QR on device (linalg.py:41-72)
    "strom_thin_svd": (C.c_int, [i64, i64, vp, vp, vp, vp, vp]),
    "strom_qr": (C.c_int, [i64, i64, vp, vp, vp, vp]),
}

EXPORTED = []
for _name, (_res, _args) in _PROTOS.items():
    _fn = getattr(lib, _name, None)
    if _fn is None:
        continue
    _fn.restype = _res
    _fn.argtypes = _args
    EXPORTED.append(_name)


def last_error() -> str:
    msg = lib.strom_last_error()
    return msg.decode() if msg else ""


_CODE_EXC = {
    1: ValueError,
    2: RuntimeError,
    3: ValueError,
    4: errors.SingularMatrixError,
    5: errors.BasisError,
    6: RuntimeError,
}


def check(rc: int, what: str = "") -> None:
    if rc:
        exc = _CODE_EXC.get(rc, RuntimeError)
        raise exc(last_error() or f"{what} failed with code {rc}")


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args), name)
