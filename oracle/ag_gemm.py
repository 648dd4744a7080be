"""CPU ORACLE for the fused AllGather + GEMM -- TEST INFRASTRUCTURE ONLY.

SURVEY.md Sec 8 row f4 ("other fused collectives: AllGather+GEMM"), PAPER.md P:180 (Sec 3.5,
"General Applicability for Collectives"): "In fully-sharded data parallel models, the
AllGather collective can be overlapped with the subsequent matrix computations", i.e. the
paper's fused-kernel principle applied to AllGather -> GEMM.  The paper gives no
formula; the computation is the plain definition of its two named steps (R#33):

    AllGather (rank-ordered):  W[s*N_r + i][k] = W_s[i][k]                    s = 0..W-1
    GEMM (a Linear layer):     Y_r[m][n]       = sum_k X_r[m][k] * W[n][k]

computed here in float64 from the bf16-exact operand values; numpy's matmul is the library
primitive for the sum (SURVEY.md Sec 8(c) allows one).  The kernel accumulates in fp32 on the
tensor cores and rounds once to the output type (R#34); ``bf16_rne`` and ``error_bound`` state
what that means for a comparison.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg may import
this module.  It shares no code with paper_2305_06942_b200/ and never imports it.
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np


def allgather_rows(shards: Sequence[np.ndarray]) -> np.ndarray:
    """P:180 AllGather of row shards, rank-ordered: shard s occupies rows s*N_r .. (s+1)*N_r."""
    K = shards[0].shape[1]
    n = sum(s.shape[0] for s in shards)
    out = np.empty((n, K), dtype=np.float64)
    row = 0
    for s in shards:
        if s.shape[1] != K:
            raise ValueError("shards disagree on K")
        out[row:row + s.shape[0], :] = s
        row += s.shape[0]
    return out


def gemm_nt(X: np.ndarray, Wfull: np.ndarray) -> np.ndarray:
    """Y[m][n] = sum_k X[m][k] * W[n][k] in float64 (the Linear layer y = x W^T)."""
    X = np.asarray(X, dtype=np.float64)
    Wfull = np.asarray(Wfull, dtype=np.float64)
    if X.shape[1] != Wfull.shape[1]:
        raise ValueError("K mismatch")
    return X @ Wfull.T


def ag_gemm(X_r: np.ndarray, shards: Sequence[np.ndarray]) -> Tuple[np.ndarray, np.ndarray]:
    """Rank r's two results: the gathered weight W and Y_r = X_r W^T (float64)."""
    Wfull = allgather_rows(shards)
    return Wfull, gemm_nt(X_r, Wfull)


def ag_gemm_entries(X_rows: np.ndarray, W_rows: np.ndarray) -> np.ndarray:
    """Sampled entries: Y[i] = sum_k X_rows[i][k] * W_rows[i][k] (one dot product per pair),
    for full-size parity on sampled (m, n) -- the caller supplies row m of X_r and row n of W."""
    return np.einsum("ik,ik->i", np.asarray(X_rows, np.float64), np.asarray(W_rows, np.float64))


def bf16_rne_bits(y: np.ndarray) -> np.ndarray:
    """Round values that are exact in fp32 to bfloat16, to nearest, ties to even (R#34); returns
    the 16-bit patterns.  NaN is not produced by the inputs here and is not handled."""
    f = np.asarray(y, dtype=np.float64).astype(np.float32)
    if not np.array_equal(f.astype(np.float64), np.asarray(y, dtype=np.float64)):
        raise ValueError("bf16_rne_bits: value not exact in fp32")
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    return ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def error_bound(X: np.ndarray, Wfull: np.ndarray, out_bits: int = 16) -> np.ndarray:
    """|Y_gpu - Y| bound per entry (R#37): fp32 accumulation of K exact products in any order,
    each add off by at most one fp32 ulp (the tensor core may truncate), gamma = 2 K 2^-24 of
    sum_k |x w|; then one rounding to the output (half an ulp: u = 2^-8 of |Y| for bf16's 8 significant
    bits, 2^-24 for fp32), taken on the accumulated value (so times (1 + gamma))."""
    K = X.shape[1]
    absdot = np.abs(np.asarray(X, np.float64)) @ np.abs(np.asarray(Wfull, np.float64)).T
    acc = 2.0 * K * 2.0 ** -24 * absdot
    out_u = 2.0 ** -8 if out_bits == 16 else 2.0 ** -24
    Y = gemm_nt(X, Wfull)
    return acc + out_u * (np.abs(Y) + acc) + 1e-30
