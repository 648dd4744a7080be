"""Device-side procedural table fill (input generation only; synth/fill.cu)."""
from __future__ import annotations

import ctypes
import os
from typing import List

import torch

from .dlrm_gen import ProblemConfig

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth_fill.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing; run __graft_entry__.build()")
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.synth_fill_table.restype = ctypes.c_int
        _lib.synth_fill_table.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int,
                                          ctypes.c_longlong, ctypes.c_ulonglong, ctypes.c_int,
                                          ctypes.c_void_p]
        _lib.synth_fill_gemm_bf16.restype = ctypes.c_int
        _lib.synth_fill_gemm_bf16.argtypes = [ctypes.c_void_p, ctypes.c_longlong,
                                              ctypes.c_longlong, ctypes.c_longlong,
                                              ctypes.c_longlong, ctypes.c_ulonglong, ctypes.c_int,
                                              ctypes.c_void_p]
    return _lib


def fill_table(dst: torch.Tensor, g: int, seed: int, mode: int) -> None:
    assert dst.is_cuda and dst.dtype == torch.float32 and dst.is_contiguous() and dst.dim() == 2
    rc = _load().synth_fill_table(dst.data_ptr(), dst.shape[0], dst.shape[1], g, seed, mode,
                                  torch.cuda.current_stream(dst.device).cuda_stream)
    if rc:
        raise RuntimeError(f"synth_fill_table failed ({rc})")


def rank_tables(cfg: ProblemConfig, r: int, device) -> List[torch.Tensor]:
    """Rank r's T_r procedural tables as views into one [T_r, R, D] device allocation."""
    T = cfg.T[r]
    big = torch.empty((max(T, 1), cfg.R, cfg.D), dtype=torch.float32, device=device)
    tabs = [big[t] for t in range(T)]
    for t, tab in enumerate(tabs):
        fill_table(tab, cfg.toff(r) + t, cfg.table_seed, cfg.value_mode)
    return tabs


def fill_gemm_bf16(dst: torch.Tensor, tensor: int, seed: int, mode: int, row0: int = 0) -> None:
    """Fill a [rows][cols] bf16 tensor with the GEMM operand generator (synth/gemm_gen.py)."""
    assert dst.is_cuda and dst.dtype == torch.bfloat16 and dst.is_contiguous() and dst.dim() == 2
    rc = _load().synth_fill_gemm_bf16(dst.data_ptr(), dst.shape[0], dst.shape[1], row0, tensor,
                                      seed, mode, torch.cuda.current_stream(dst.device).cuda_stream)
    if rc:
        raise RuntimeError(f"synth_fill_gemm_bf16 failed ({rc})")
