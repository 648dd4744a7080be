"""Python binding of the fused AllGather + GEMM (include/ag_gemm.h; SURVEY.md Sec 8 row f4,
PAPER.md P:180).  Argument marshalling only: the gather, the flags and the GEMM all run in
``ag_gemm_kernel`` (csrc/ag_gemm.cu); there is no CPU or library fallback.

    h = AgGemm(rank, W, device, allgather)        # one rank (torch_allgather / LocalGroup)
    h.register(M, n_local, K)                     # collective
    Y, Wg = h.forward(X, w_local)                 # collective: Y = X @ AllGather(w)^T

``AgGemmLoopback`` drives W virtual ranks on one device (W handles, W streams, grid divided W
ways so every rank's persistent kernel is resident while it waits for its peers' chunks).
"""
from __future__ import annotations

import ctypes
import traceback
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import lib
from .emb_a2a import AllgatherFn, EmbA2AError, LocalGroup, _stream_ptr, _view, run_ranks


class AgGemm:
    def __init__(self, rank: int, world_size: int, device, allgather: Optional[AllgatherFn],
                 options: Optional[dict] = None):
        self.device = torch.device(device) if not isinstance(device, torch.device) else device
        if self.device.type != "cuda":
            raise ValueError("AgGemm runs on CUDA devices only (no CPU fallback)")
        self.rank, self.W = rank, world_size
        self._ag = allgather
        self._cb = _lib.ALLGATHER_FN(self._trampoline)
        self._h = ctypes.c_void_p()
        rc = lib.ag_gemm_init(rank, world_size, self.device.index or 0, self._cb, None,
                              ctypes.byref(self._h))
        if rc:
            raise EmbA2AError(rc, "ag_gemm_init")
        self.shape = None
        for k, v in (options or {}).items():
            self.set_option(k, v)

    def _trampoline(self, send, recv, nbytes, user):
        try:
            out = self._ag(ctypes.string_at(send, nbytes))
            if len(out) != self.W * nbytes:
                raise ValueError("all-gather returned the wrong size")
            ctypes.memmove(recv, out, len(out))
            return 0
        except Exception:
            traceback.print_exc()
            return 1

    def _err(self, rc: int, what: str):
        if rc:
            raise EmbA2AError(rc, what, lib.ag_gemm_last_error(self._h).decode())

    def register(self, M: int, n_local: int, K: int, out_dtype=torch.bfloat16) -> None:
        if out_dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("out_dtype: torch.bfloat16 or torch.float32")
        f32 = 1 if out_dtype == torch.float32 else 0
        self._err(lib.ag_gemm_register(self._h, M, n_local, K, f32), "ag_gemm_register")
        self.shape = (M, n_local, K)
        self.out_dtype = out_dtype

    def forward(self, X: torch.Tensor, w_local: torch.Tensor, Y: Optional[torch.Tensor] = None,
                stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
        """Y = X @ AllGather(w)^T (collective).  Returns (Y, gathered-weight view [N][K] bf16,
        valid until this rank's next forward)."""
        M, Nr, K = self.shape
        N = self.W * Nr
        for t, shp, name in ((X, (M, K), "X"), (w_local, (Nr, K), "w_local")):
            if (t.device != self.device or t.dtype != torch.bfloat16 or not t.is_contiguous()
                    or tuple(t.shape) != shp):
                raise ValueError(f"{name} must be a contiguous bf16 {shp} tensor on {self.device}")
        if Y is None:
            Y = torch.empty((M, N), dtype=self.out_dtype, device=self.device)
        elif Y.device != self.device or Y.dtype != self.out_dtype or not Y.is_contiguous() \
                or tuple(Y.shape) != (M, N):
            raise ValueError(f"Y must be a contiguous {self.out_dtype} ({M}, {N}) tensor")
        wg = ctypes.c_void_p()
        self._err(lib.ag_gemm_forward(self._h, X.data_ptr(), w_local.data_ptr(), Y.data_ptr(),
                                      _stream_ptr(stream, self.device), ctypes.byref(wg)),
                  "ag_gemm_forward")
        return Y, _view(wg.value or 0, (N, K), self.device, torch.bfloat16)

    def set_option(self, key: str, value: int) -> None:
        self._err(lib.ag_gemm_set_option(self._h, key.encode(), int(value)), f"set_option({key})")

    def get_option(self, key: str) -> int:
        v = ctypes.c_int64()
        self._err(lib.ag_gemm_get_option(self._h, key.encode(), ctypes.byref(v)), "get_option")
        return v.value

    def query(self, key: str) -> int:
        v = ctypes.c_int64()
        self._err(lib.ag_gemm_query(self._h, key.encode(), ctypes.byref(v)), f"query({key})")
        return v.value

    def read_flags(self) -> np.ndarray:
        n = self.W * self.query("chunks")
        out = np.zeros(max(n, 1), dtype=np.uint32)
        got = ctypes.c_int64()
        self._err(lib.ag_gemm_read_flags(self._h, out.ctypes.data, out.size, ctypes.byref(got)),
                  "read_flags")
        return out[:n].reshape(self.W, -1)

    def check(self) -> None:
        self._err(lib.ag_gemm_check(self._h), "ag_gemm_check")

    def status(self) -> int:
        """The asynchronous error status without raising (0 = OK)."""
        return int(lib.ag_gemm_check(self._h))

    def destroy(self) -> None:
        if self._h:
            lib.ag_gemm_destroy(self._h)
            self._h = ctypes.c_void_p()


class AgGemmLoopback:
    """W virtual ranks of the fused AllGather + GEMM on ONE device."""

    def __init__(self, world_size: int, device="cuda:0", options: Optional[dict] = None):
        self.W = world_size
        self.device = torch.device(device)
        self.group = LocalGroup(world_size)
        self.handles: List[AgGemm] = [
            AgGemm(r, world_size, self.device, self.group.allgather_for(r), options)
            for r in range(world_size)]
        self.streams = [torch.cuda.Stream(self.device) for _ in range(world_size)]

    def set_option(self, key: str, value: int) -> None:
        for h in self.handles:
            h.set_option(key, value)

    def register(self, M: int, n_local: int, K: int, out_dtype=torch.bfloat16) -> None:
        run_ranks(lambda r: self.handles[r].register(M, n_local, K, out_dtype), self.W)

    def forward(self, X: Sequence[torch.Tensor], w: Sequence[torch.Tensor],
                Y: Optional[Sequence[torch.Tensor]] = None, sync: bool = True):
        cur = torch.cuda.current_stream(self.device)
        for s in self.streams:
            s.wait_stream(cur)
        outs = [h.forward(X[r], w[r], None if Y is None else Y[r], stream=self.streams[r])
                for r, h in enumerate(self.handles)]
        for s in self.streams:
            cur.wait_stream(s)
        if sync:
            torch.cuda.synchronize(self.device)
            for h in self.handles:
                h.check()
        return outs

    def destroy(self) -> None:
        run_ranks(lambda r: self.handles[r].destroy(), self.W)
