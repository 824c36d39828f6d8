"""ctypes binding of libtls_b200.so (the C ABI in include/tls_b200.h).

The shared library is built in-tree (``__graft_entry__.build()`` or
``python -m paper_2401_03915_b200.build``).  There is no fallback: if the
library is missing or no CUDA device is present, every GPU entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtls_b200.so")

TLS_OK = 0
TLS_ERR_DIM = 1
TLS_ERR_BREAKDOWN = 2
TLS_ERR_SUBDOMAIN = 3
TLS_ERR_COARSE = 4
TLS_ERR_CAP = 5
TLS_ERR_ARG = 6
TLS_ERR_STATE = 7
TLS_ERR_CUDA = 8
TLS_ERR_OOM = 9
TLS_ERR_FORMAT = 10
TLS_ERR_IO = 11
TLS_ERR_CALLBACK = 12

ONE_LEVEL = {"asm": 0, "ras": 1}
COMBINE = {"none": 0, "additive": 1, "deflated": 2}


class TlsStatus(C.Structure):
    _fields_ = [("code", C.c_int32), ("iterations", C.c_int32), ("converged", C.c_int32),
                ("iteration", C.c_int32), ("value", C.c_double), ("gpu_launches", C.c_int32),
                ("pad_", C.c_int32)]


ITER_CB = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_double))

_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double

# name -> (restype, argtypes); every symbol declared in include/tls_b200.h
SIGNATURES = {
    "tls_abi_version": (_I32, []),
    "tls_ctx_create": (_I32, [_I32, C.POINTER(_P)]),
    "tls_ctx_destroy": (None, [_P]),
    "tls_ctx_last_error": (C.c_char_p, [_P]),
    "tls_ctx_device_bytes": (_I64, [_P]),
    "tls_matrix_upload": (_I32, [_P, _I64, _I64, _P, _P, _P, _I32]),
    "tls_spmv": (_I32, [_P, _P, _P, _P]),
    "tls_subdomains_upload": (_I32, [_P, _I32, _P, _P, _P]),
    "tls_subdomain_max_size": (_I32, [_P]),
    "tls_extract_blocks": (_I32, [_P, _I32, _I32, _P, _I64, _P]),
    "tls_store_local_inverse": (_I32, [_P, _I32, _I32, _P, _I64, _P]),
    "tls_coarse_upload": (_I32, [_P, _I32, _P, _P, _P, _P]),
    "tls_precond_finalize": (_I32, [_P, _I32, _I32]),
    "tls_precond_apply": (_I32, [_P, _P, _P, _P]),
    "tls_apply_one_level": (_I32, [_P, _P, _P, _P]),
    "tls_coarse_apply": (_I32, [_P, _P, _P, _P]),
    "tls_coarse_refine": (_I32, [_P, _P, _P]),
    "tls_coarse_chain": (_I32, [_P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _I64, _P]),
    "tls_local_solve": (_I32, [_P, _P, _I32, _P, _P, _P]),
    "tls_coarse_restrict": (_I32, [_P, _P, _P, _P]),
    "tls_coarse_solve": (_I32, [_P, _P, _P, _P]),
    "tls_coarse_prolong": (_I32, [_P, _P, _P, _P]),
    "tls_pcg": (_I32, [_P, _P, _P, _D, _I32, _I32, _P, _P, C.POINTER(TlsStatus), ITER_CB, _P, _P]),
    "tls_gmres": (_I32, [_P, _P, _P, _D, _I32, _I32, _I32, _P, C.POINTER(TlsStatus), ITER_CB, _P, _P]),
    "tls_report": (_I32, [_P, C.POINTER(_I64), C.POINTER(_I32), C.POINTER(_I32), C.POINTER(_I64)]),
    "tls_profile_local_solve": (_I32, [_P, _I32, C.POINTER(_D), C.POINTER(_D), _P]),
    "tls_set_kernel_timing": (_I32, [_P, _I32]),
    "tls_kernel_timing": (_I32, [_P, C.POINTER(_D), C.POINTER(_I64)]),
    "tls_set_owned_range": (_I32, [_P, _I32, _I32]),
    "tls_set_row_partition": (_I32, [_P, _I64, _P, _I32, _P, _I32]),
    "tls_set_halo": (_I32, [_P, _I32, _P, _P, _P, _P, _P]),
    "tls_set_remote_contrib": (_I32, [_P, _I32, _P, _P, _P, _P]),
    "tls_set_local_kind": (_I32, [_P, _I32]),
    "tls_band_cholesky": (_I32, [_P, _I64, _I32, _P, _I32, _P, _P, _P]),
    "tls_mm_parse": (_I32, [C.c_char_p, _I64, _I32, C.POINTER(_P)]),
    "tls_mm_load": (_I32, [C.c_char_p, _I32, C.POINTER(_P)]),
    "tls_mm_info": (_I32, [_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I32),
                           C.POINTER(_I64), C.POINTER(C.c_char_p)]),
    "tls_mm_export": (_I32, [_P, _P, _P, _P]),
    "tls_mm_free": (None, [_P]),
    "tls_mm_write": (_I32, [C.c_char_p, _I64, _I64, _P, _P, _P, _I32]),
    "tls_store_local_band": (_I32, [_P, _I32, _I32, _P, _I64, _P, _I32, _P, _P, _P]),
    "tls_store_local_band_lu": (_I32, [_P, _I32, _I32, _P, _I64, _P, _P, _I32, _P, _P, _P, _P, _P]),
    "tls_nccl_unique_id": (_I32, [_P, _I32]),
    "tls_comm_init_nccl": (_I32, [_P, _P, _I32, _I32]),
    "tls_group_create": (_I32, [_I32, C.POINTER(_P)]),
    "tls_group_destroy": (None, [_P]),
    "tls_comm_init_group": (_I32, [_P, _P, _I32]),
    "tls_comm_init_record": (_I32, [_P, _I32, _I32]),
    "tls_comm_record_log": (_I64, [_P, _P, _I64]),
    "tls_comm_info": (_I32, [_P, _P]),
    "tls_coarse_info": (_I32, [_P, _P]),
    "tls_coarse_basis_fetch": (_I32, [_P, _P, _I64]),
    "tls_set_coarse_layout": (_I32, [_P, _I32, _P]),
    "tls_graph_build": (_I32, [_P, C.POINTER(_I64)]),
    "tls_graph_fetch": (_I32, [_P, _P, _P]),
    "tls_overlap_build": (_I32, [_P, _I32, _P, _I32, C.POINTER(_I64), C.POINTER(_I32)]),
    "tls_overlap_fetch": (_I32, [_P, _P, _P, _P, _P]),
    "tls_graph_release": (_I32, [_P]),
    "tls_syevj_batched": (_I32, [_P, _I64, _I32, _P, _P, _P]),
    "tls_svdj_batched": (_I32, [_P, _I64, _I32, _I32, _P, _P, _P]),
    "tls_perm_lower": (_I32, [_P, _P, _P, _P, _I32, _I64, _P]),
    "tls_set_kernel_trace": (_I32, [_P, _I32]),
    "tls_kernel_trace_dump": (_I64, [_P, _P, _I64]),
    "tls_band_solve_multi": (_I32, [_P, _I64, _I32, _P, _P, _I32, _P, _I64, _P]),
    "tls_band_lu": (_I32, [_P, _I64, _I32, _P, _P, _I32, _P, _P, _P]),
    "tls_galerkin_assemble": (_I32, [_P, _P, _I64, _P, _P, _P, _P, _I32, _P, _P, _I64, _P, _I64, _P]),
    "tls_rank_filter_pivots": (_I32, [_P, _P, _P, _P, _I32, _P, _P, _P]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def load(path=LIB_PATH):
    """Load the in-tree shared library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryMissing(f"{path} not built; run __graft_entry__.build()")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def ptr(t):
    """Raw device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        if not t.is_contiguous():
            raise ValueError("raw pointers need C-contiguous (row-major) tensors")
        return C.c_void_p(t.data_ptr())
    if not t.flags["C_CONTIGUOUS"]:
        raise ValueError("raw pointers need C-contiguous arrays")
    return C.c_void_p(t.ctypes.data)
