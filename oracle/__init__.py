"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain single-threaded C (oracle/oracle.c) behind a ctypes wrapper.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` leg may import
this package.  It shares no code with paper_2305_06942_b200/ and never imports it.

Every function cites the passage it follows (see oracle.c's header for the full map):
  emb_a2a            P:119 (sum pooling), P:145 (contiguous batch blocks), P:147 (layout)
  emb_a2a_rows       same definition, selected rows, procedural tables
  destination
  slice_plan         P:145; S:103, S:144
  signal_count
  table_value        input generator, not the method
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
GCC_FLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c99"]

OK, EINVAL, EINDEX, ECAP = 0, 1, 8, 9


class OracleError(RuntimeError):
    def __init__(self, rc: int, what: str):
        names = {EINVAL: "EINVAL", EINDEX: "EINDEX (index out of range, S:113)", ECAP: "ECAP"}
        super().__init__(f"oracle {what}: {names.get(rc, rc)}")
        self.rc = rc


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with plain gcc (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", _LIB + ".tmp", _SRC])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.oracle_splitmix64.restype = ctypes.c_uint64
        L.oracle_splitmix64.argtypes = [ctypes.c_uint64]
        L.oracle_table_value.restype = ctypes.c_float
        L.oracle_table_value.argtypes = [ctypes.c_uint64, I32, I64, I64, I64]
        L.oracle_destination.restype = I32
        L.oracle_destination.argtypes = [I32, P, I64, P, P]
        L.oracle_emb_a2a.restype = I32
        L.oracle_emb_a2a.argtypes = [I32, P, I32, I64, P, P, P, P, P, P, I32, P]
        L.oracle_emb_a2a_rows.restype = I32
        L.oracle_emb_a2a_rows.argtypes = [ctypes.c_uint64, I32, I32, P, I32, I64, P, P, P, P, P,
                                          I32, P, I64, I32, P, I32]
        L.oracle_emb_a2a_ex.restype = I32
        L.oracle_emb_a2a_ex.argtypes = [I32, P, I32, I64, P, P, I32, P, P, P, P, P, I32, I32, P]
        L.oracle_emb_a2a_rows_ex.restype = I32
        L.oracle_emb_a2a_rows_ex.argtypes = [ctypes.c_uint64, I32, I32, P, I32, I64, P, P, P, P, P,
                                             P, I32, I32, P, I64, I32, P, I32]
        L.oracle_bf16_to_float.restype = ctypes.c_float
        L.oracle_bf16_to_float.argtypes = [ctypes.c_uint16]
        L.oracle_f16_to_float.restype = ctypes.c_float
        L.oracle_f16_to_float.argtypes = [ctypes.c_uint16]
        L.oracle_round_to_half.restype = ctypes.c_uint16
        L.oracle_round_to_half.argtypes = [ctypes.c_float, I32]
        L.oracle_round_array.restype = None
        L.oracle_round_array.argtypes = [P, P, I64, I32]
        L.oracle_backward_sgd.restype = I32
        L.oracle_backward_sgd.argtypes = [I32, P, I32, I64, P, P, P, P, P, P, P, I32, P,
                                          ctypes.c_float]
        L.oracle_slice_plan.restype = I32
        L.oracle_slice_plan.argtypes = [I32, I32, P, I32, I64, I32, P, I64, P]
        L.oracle_signal_count.restype = I64
        L.oracle_signal_count.argtypes = [I32, I32, P, P, I64]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _ptr_array(arrs: Sequence[np.ndarray]) -> np.ndarray:
    return np.array([a.ctypes.data for a in arrs], dtype=np.uintp)


def splitmix64(x: int) -> int:
    return int(lib().oracle_splitmix64(x))


def table_value(seed: int, mode: int, g: int, row: int, d: int) -> float:
    return float(lib().oracle_table_value(seed, mode, g, row, d))


def destination(W: int, part: Sequence[int], j: int) -> Tuple[int, int]:
    """(s, i): destination rank and local row of global sample j."""
    p = np.ascontiguousarray(part, dtype=np.int64)
    s = ctypes.c_int(0)
    i = ctypes.c_int64(0)
    rc = lib().oracle_destination(W, _ptr(p), j, ctypes.addressof(s), ctypes.addressof(i))
    if rc:
        raise OracleError(rc, "destination")
    return s.value, i.value


def _common(part, T, indices, offsets):
    p = np.ascontiguousarray(part, dtype=np.int64)
    Ta = np.ascontiguousarray(T, dtype=np.int32)
    idx = [np.ascontiguousarray(a, dtype=np.int32) for a in indices]
    off = [np.ascontiguousarray(a, dtype=np.int32) for a in offsets]
    nnz = np.array([a.size for a in idx], dtype=np.int64)
    # keep non-empty buffers so ctypes pointers are valid
    idx = [a if a.size else np.zeros(1, dtype=np.int32) for a in idx]
    return p, Ta, idx, off, nnz


F32, BF16, F16 = 0, 1, 2
SUM, MEAN = 0, 1


def round_to_half(a: np.ndarray, dtype: int) -> np.ndarray:
    """16-bit output (R#32): float32 values -> bfloat16 (BF16) or binary16 (F16) bits, rounded
    to nearest, ties to even, once (oracle.c oracle_round_to_half)."""
    x = np.ascontiguousarray(a, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.uint16)
    if x.size:
        lib().oracle_round_array(_ptr(x), _ptr(out), x.size, dtype)
    return out


def bf16_to_float(bits: int) -> float:
    return float(lib().oracle_bf16_to_float(bits))


def f16_to_float(bits: int) -> float:
    return float(lib().oracle_f16_to_float(bits))


def _weights(weights, idx):
    if weights is None:
        return None, None
    w = [np.ascontiguousarray(a, dtype=np.float32) for a in weights]
    w = [a if a.size else np.zeros(1, dtype=np.float32) for a in w]
    arr = _ptr_array(w)
    return w, arr


def emb_a2a(part: Sequence[int], D: int, B: int, T: Sequence[int], tables: Sequence[np.ndarray],
            indices: Sequence[np.ndarray], offsets: Sequence[np.ndarray],
            precision: int = 32, dtype: int = F32, weights: Optional[Sequence[np.ndarray]] = None,
            pooling: int = SUM, out_dtype: int = F32) -> List[np.ndarray]:
    """The plain definition over materialised tables (G arrays [rows_g, D]).

    dtype F32: float32 tables; BF16 / F16: uint16 arrays holding bfloat16 / binary16 bits.
    weights: optional per-rank per-sample weights aligned with indices (sum pooling only).
    pooling: SUM or MEAN (P:119 ..._sum_mean).
    out_dtype: F32, or BF16 / F16 for a 16-bit output: the fp32 result rounded once, to nearest
    even (R#32) -- returned as uint16 bit arrays.
    Returns out_s for every destination rank s: [b_s, G*D], float32 (precision=32) or float64.
    """
    W = len(T)
    p, Ta, idx, off, nnz = _common(part, T, indices, offsets)
    edt = np.float32 if dtype == F32 else np.uint16
    tabs = [np.ascontiguousarray(t, dtype=edt) for t in tables]
    rows = np.array([t.shape[0] for t in tabs], dtype=np.int64)
    G = int(Ta.sum())
    assert len(tabs) == G
    dt = np.float64 if precision == 64 else np.float32
    outs = [np.full((int(p[s + 1] - p[s]), G * D), np.nan, dtype=dt) for s in range(W)]
    outs_keep = [o if o.size else np.zeros(1, dtype=dt) for o in outs]
    wk, warr = _weights(weights, idx)
    keep = [_ptr_array(tabs), _ptr_array(idx), _ptr_array(off), _ptr_array(outs_keep)]
    rc = lib().oracle_emb_a2a_ex(W, _ptr(p), D, B, _ptr(Ta), _ptr(keep[0]), dtype, _ptr(rows),
                                 _ptr(keep[1]), _ptr(keep[2]),
                                 _ptr(warr) if warr is not None else None, _ptr(nnz), pooling,
                                 precision, _ptr(keep[3]))
    if rc:
        raise OracleError(rc, "emb_a2a")
    if out_dtype != F32:
        assert precision == 32
        return [round_to_half(o, out_dtype) for o in outs]
    return outs


def emb_a2a_rows(seed: int, mode: int, part: Sequence[int], D: int, B: int, T: Sequence[int],
                 R: int, indices: Sequence[np.ndarray], offsets: Sequence[np.ndarray], s: int,
                 rows_i: Sequence[int], precision: int = 32, check_inputs: bool = True,
                 weights: Optional[Sequence[np.ndarray]] = None, pooling: int = SUM,
                 out_dtype: int = F32) -> np.ndarray:
    """Selected rows of out_s with procedural tables (every table has R rows); out_dtype as in
    emb_a2a (16-bit outputs come back as uint16 bits)."""
    W = len(T)
    p, Ta, idx, off, nnz = _common(part, T, indices, offsets)
    G = int(Ta.sum())
    rows = np.full(G, R, dtype=np.int64)
    sel = np.ascontiguousarray(rows_i, dtype=np.int64)
    dt = np.float64 if precision == 64 else np.float32
    out = np.full((max(sel.size, 1), G * D), np.nan, dtype=dt)
    keep = [_ptr_array(idx), _ptr_array(off), sel if sel.size else np.zeros(1, np.int64)]
    wk, warr = _weights(weights, idx)
    rc = lib().oracle_emb_a2a_rows_ex(seed, mode, W, _ptr(p), D, B, _ptr(Ta), _ptr(rows),
                                      _ptr(keep[0]), _ptr(keep[1]),
                                      _ptr(warr) if warr is not None else None, _ptr(nnz),
                                      pooling, s, _ptr(keep[2]), sel.size, precision, _ptr(out),
                                      int(check_inputs))
    if rc:
        raise OracleError(rc, "emb_a2a_rows")
    if out_dtype != F32:
        assert precision == 32
        return round_to_half(out[: sel.size], out_dtype)
    return out[: sel.size]


def backward_sgd(part: Sequence[int], D: int, B: int, T: Sequence[int],
                 tables: Sequence[np.ndarray], indices: Sequence[np.ndarray],
                 offsets: Sequence[np.ndarray], grad: Sequence[np.ndarray], lr: float,
                 weights: Optional[Sequence[np.ndarray]] = None, pooling: int = SUM
                 ) -> List[np.ndarray]:
    """Backward + SGD (f3): returns updated copies of the G fp32 tables.  grad[s] is destination
    rank s's pooled-output gradient [b_s, G*D] (the forward output's layout)."""
    W = len(T)
    p, Ta, idx, off, nnz = _common(part, T, indices, offsets)
    tabs = [np.array(t, dtype=np.float32, copy=True, order="C") for t in tables]
    rows = np.array([t.shape[0] for t in tabs], dtype=np.int64)
    grads = [np.ascontiguousarray(x, dtype=np.float32) for x in grad]
    grads = [x if x.size else np.zeros(1, np.float32) for x in grads]
    wk, warr = _weights(weights, idx)
    keep = [_ptr_array(tabs), _ptr_array(idx), _ptr_array(off), _ptr_array(grads)]
    rc = lib().oracle_backward_sgd(W, _ptr(p), D, B, _ptr(Ta), _ptr(keep[0]), _ptr(rows),
                                   _ptr(keep[1]), _ptr(keep[2]),
                                   _ptr(warr) if warr is not None else None, _ptr(nnz), pooling,
                                   _ptr(keep[3]), lr)
    if rc:
        raise OracleError(rc, "backward_sgd")
    return tabs


def slice_plan(r: int, W: int, part: Sequence[int], T_r: int, S: int, order: int = 0) -> np.ndarray:
    """Rank r's slices in issue order: int32 [n, 4] = (s, t, i0, nb)."""
    p = np.ascontiguousarray(part, dtype=np.int64)
    n = ctypes.c_int64(0)
    cap = 1
    while True:
        out = np.zeros((cap, 4), dtype=np.int32)
        rc = lib().oracle_slice_plan(r, W, _ptr(p), T_r, S, order, _ptr(out), cap,
                                     ctypes.addressof(n))
        if rc == ECAP:
            cap = n.value
            continue
        if rc:
            raise OracleError(rc, "slice_plan")
        return out[: n.value]


def signal_count(src: int, dst: int, T: Sequence[int], part: Sequence[int], S: int) -> int:
    Ta = np.ascontiguousarray(T, dtype=np.int32)
    p = np.ascontiguousarray(part, dtype=np.int64)
    return int(lib().oracle_signal_count(src, dst, _ptr(Ta), _ptr(p), S))
