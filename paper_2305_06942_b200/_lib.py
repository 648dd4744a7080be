"""ctypes view of libemba2a.so (include/emb_a2a.h).  Argument marshalling only.

The library is built in-tree by ``__graft_entry__.build()``.  There is no fallback: if the
shared object is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EMBA2A_LIB") or os.path.join(_HERE, "libemba2a.so")

OK, EINVAL, ESTATE, ECUDA, ENOMEM, EPEER, EBOOT, ETIMEOUT, EINDEX = range(9)
F32, BF16, F16 = 0, 1, 2          # emb_a2a_dtype
SUM, MEAN = 0, 1                  # emb_a2a_pooling
MAX_WORLD = 64

ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                ctypes.c_void_p)

if not os.path.exists(LIB_PATH):
    raise RuntimeError(
        f"{LIB_PATH} is missing: the CUDA library has not been built "
        "(run `python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")

lib = ctypes.CDLL(LIB_PATH)

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_PI64 = ctypes.POINTER(ctypes.c_int64)

_SIGS = {
    "emb_a2a_abi_version": (_I, []),
    "emb_a2a_status_string": (ctypes.c_char_p, [_I]),
    "emb_a2a_last_error": (ctypes.c_char_p, [_P]),
    "emb_a2a_init": (_I, [_I, _I, _I, ALLGATHER_FN, _P, ctypes.POINTER(_P)]),
    "emb_a2a_register_tables": (_I, [_P, _I, _P, _P, _I, _I64, _P]),
    "emb_a2a_register_tables_ex": (_I, [_P, _I, _P, _P, _I, _I, _I, _I64, _P]),
    "emb_a2a_forward": (_I, [_P, _P, _P, _I64, _P, ctypes.POINTER(_P), _PI64, _PI64]),
    "emb_a2a_forward_weighted": (_I, [_P, _P, _P, _P, _I64, _P, ctypes.POINTER(_P), _PI64, _PI64]),
    "emb_a2a_forward_host": (_I, [_P, _P, _P, _I64, _P, _P]),
    "emb_a2a_forward_host_batch": (_I, [_P, _I, _P, _P, _P, _P, _P]),
    "emb_a2a_pool_local": (_I, [_P, _P, _P, _I64, _P, _P]),
    "emb_a2a_pool_local_weighted": (_I, [_P, _P, _P, _P, _I64, _P, _P]),
    "emb_a2a_backward_plan": (_I, [_P, _P, _P, _P, _I64, _P]),
    "emb_a2a_backward": (_I, [_P, _P, ctypes.c_float, _P]),
    "emb_a2a_backward_local": (_I, [_P, _P, ctypes.c_float, _P]),
    "emb_a2a_device_barrier": (_I, [_P, _P]),
    "emb_a2a_peer_store_probe": (_I, [_P, _I64, _P, _PI64]),
    "emb_a2a_check": (_I, [_P]),
    "emb_a2a_set_option": (_I, [_P, ctypes.c_char_p, _I64]),
    "emb_a2a_get_option": (_I, [_P, ctypes.c_char_p, _PI64]),
    "emb_a2a_query": (_I, [_P, ctypes.c_char_p, _PI64]),
    "emb_a2a_slice_plan": (_I, [_P, _P, _I64, _PI64]),
    "emb_a2a_read_flags": (_I, [_P, _P, _I]),
    "emb_a2a_read_trace": (_I, [_P, _P, _I64, _PI64]),
    "emb_a2a_destroy": (_I, [_P]),
}

EXPORTED = tuple(_SIGS)

# include/ag_gemm.h: the fused AllGather + GEMM
_AG_SIGS = {
    "ag_gemm_init": (_I, [_I, _I, _I, ALLGATHER_FN, _P, ctypes.POINTER(_P)]),
    "ag_gemm_register": (_I, [_P, _I64, _I64, _I64, _I]),
    "ag_gemm_forward": (_I, [_P, _P, _P, _P, _P, ctypes.POINTER(_P)]),
    "ag_gemm_set_option": (_I, [_P, ctypes.c_char_p, _I64]),
    "ag_gemm_get_option": (_I, [_P, ctypes.c_char_p, _PI64]),
    "ag_gemm_query": (_I, [_P, ctypes.c_char_p, _PI64]),
    "ag_gemm_read_flags": (_I, [_P, _P, _I64, _PI64]),
    "ag_gemm_check": (_I, [_P]),
    "ag_gemm_destroy": (_I, [_P]),
    "ag_gemm_last_error": (ctypes.c_char_p, [_P]),
}
AG_EXPORTED = tuple(_AG_SIGS)
_SIGS_ALL = dict(_SIGS, **_AG_SIGS)

for _name, (_res, _args) in _SIGS_ALL.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

if lib.emb_a2a_abi_version() != 1:
    raise RuntimeError("libemba2a.so ABI version mismatch")


def status_string(rc: int) -> str:
    return lib.emb_a2a_status_string(rc).decode()
