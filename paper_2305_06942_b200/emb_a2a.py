"""Python binding of the fused EmbeddingBag(sum) + All-to-All (thin; marshalling only).

Every step of the forward runs in libemba2a.so's sm_100a kernels (include/emb_a2a.h).  Torch
supplies device memory, streams and -- for the one-off bootstrap all-gather of buffer handles --
the process group.  Method: arXiv 2305.06942, Sec 3.2-3.3.
"""
from __future__ import annotations

import ctypes
import threading
import traceback
from typing import Callable, List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import lib

AllgatherFn = Callable[[bytes], bytes]     # rank's bytes -> W * len(bytes), rank-ordered


class EmbA2AError(RuntimeError):
    def __init__(self, status: int, what: str, detail: str = ""):
        super().__init__(f"{what}: {_lib.status_string(status)}" + (f" ({detail})" if detail else ""))
        self.status = status


# ------------------------------------------------------------------------ bootstrap channels

class LocalGroup:
    """In-process all-gather for W virtual ranks driven from W host threads (loopback on one
    device).  ``allgather_for(r)`` returns rank r's callable."""

    def __init__(self, world_size: int, timeout: float = 120.0):
        self.W = world_size
        self._slots: List[Optional[bytes]] = [None] * world_size
        self._b1 = threading.Barrier(world_size, timeout=timeout)
        self._b2 = threading.Barrier(world_size, timeout=timeout)

    def allgather_for(self, rank: int) -> AllgatherFn:
        def f(data: bytes) -> bytes:
            self._slots[rank] = data
            self._b1.wait()
            out = b"".join(self._slots)      # type: ignore[arg-type]
            self._b2.wait()
            return out
        return f


def torch_allgather(group=None, device: Optional[torch.device] = None) -> AllgatherFn:
    """All-gather over a torch.distributed process group (gloo: CPU tensors; nccl: device)."""
    import torch.distributed as dist

    def f(data: bytes) -> bytes:
        W = dist.get_world_size(group)
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()))
        outs = [torch.empty_like(t) for _ in range(W)]
        dist.all_gather(outs, t, group=group)
        return torch.cat(outs).cpu().numpy().tobytes()
    return f


# ------------------------------------------------------------------------ device views

class _CudaView:
    """__cuda_array_interface__ over library-owned device memory (zero-copy torch view)."""

    def __init__(self, ptr: int, shape, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2, "strides": None}


def _view(ptr: int, shape, device: torch.device, dtype=torch.float32) -> torch.Tensor:
    n = int(np.prod(shape)) if len(shape) else 1
    if n == 0 or ptr == 0:
        return torch.empty(tuple(shape), dtype=dtype, device=device)
    if dtype == torch.float32:
        return torch.as_tensor(_CudaView(ptr, shape), device=device)
    # 16-bit outputs: __cuda_array_interface__ has no bfloat16 typestr; view the bits
    return torch.as_tensor(_CudaView(ptr, shape, "<i2"), device=device).view(dtype)


def _stream_ptr(stream, device) -> int:
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return int(stream.cuda_stream)


def _check_dev_tensor(t: torch.Tensor, dtype, name: str, device):
    if t.device != device or t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor on {device}")


# ------------------------------------------------------------------------ the handle

class EmbA2A:
    """One rank's handle.  Collective calls (register_tables, forward, forward_host, destroy) must
    be made by every rank in the same order."""

    def __init__(self, rank: int, world_size: int, device, allgather: AllgatherFn,
                 options: Optional[dict] = None):
        self.device = torch.device(device) if not isinstance(device, torch.device) else device
        if self.device.type != "cuda":
            raise ValueError("EmbA2A runs on CUDA devices only (no CPU fallback)")
        self.rank, self.W = rank, world_size
        self._ag = allgather
        self._cb = _lib.ALLGATHER_FN(self._trampoline)
        self._h = ctypes.c_void_p()
        rc = lib.emb_a2a_init(rank, world_size, self.device.index or 0, self._cb, None,
                              ctypes.byref(self._h))
        if rc:
            raise EmbA2AError(rc, "emb_a2a_init")
        self._tables: List[torch.Tensor] = []
        self._views = {}          # (ptr, rows, cols) -> cached zero-copy view of a recv buffer
        self._stream_cache = None
        for k, v in (options or {}).items():
            self.set_option(k, v)

    # called from C (any thread) inside init / register / destroy
    def _trampoline(self, send, recv, nbytes, user):
        try:
            data = ctypes.string_at(send, nbytes)
            out = self._ag(data)
            if len(out) != self.W * nbytes:
                raise ValueError("all-gather returned the wrong size")
            ctypes.memmove(recv, out, len(out))
            return 0
        except Exception:      # the C side turns this into EMB_A2A_EBOOT
            traceback.print_exc()
            return 1

    def _err(self, rc: int, what: str):
        if rc:
            detail = lib.emb_a2a_last_error(self._h).decode(errors="replace") if self._h else ""
            raise EmbA2AError(rc, what, detail)

    # -------------------------------------------------------------- collective API
    _DTYPES = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16, torch.float16: _lib.F16}

    def register_tables(self, tables: Sequence[torch.Tensor], global_batch: int,
                        partition: Optional[Sequence[int]] = None, pooling: str = "sum",
                        dtype: Optional[torch.dtype] = None) -> None:
        """tables: this rank's T_r [rows, D] device tensors, float32 / bfloat16 / float16 (kept
        alive by the handle).  pooling: "sum" or "mean".  dtype: only needed when this
        rank registers no tables (must match the other ranks)."""
        tabs = list(tables)
        D = int(tabs[0].shape[1]) if tabs else int(self._dim_hint)
        tdt = tabs[0].dtype if tabs else (dtype or torch.float32)
        if tdt not in self._DTYPES:
            raise ValueError(f"unsupported table dtype {tdt}")
        for t in tabs:
            _check_dev_tensor(t, tdt, "table", self.device)
            if t.dim() != 2 or t.shape[1] != D:
                raise ValueError("tables must be [rows, D] with one D and one dtype")
        self._tables = tabs
        ptrs = (ctypes.c_void_p * max(1, len(tabs)))(*[t.data_ptr() for t in tabs])
        rows = (ctypes.c_int64 * max(1, len(tabs)))(*[t.shape[0] for t in tabs])
        part = None
        if partition is not None:
            part = (ctypes.c_int64 * (self.W + 1))(*[int(x) for x in partition])
        pool = {"sum": _lib.SUM, "mean": _lib.MEAN}[pooling]
        rc = lib.emb_a2a_register_tables_ex(self._h, len(tabs), ptrs, rows, D, self._DTYPES[tdt],
                                            pool, int(global_batch), part)
        self._err(rc, "emb_a2a_register_tables")
        self._views = {}
        self._fwd_out = (ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64())
        self._fwd_refs = tuple(ctypes.byref(x) for x in self._fwd_out)
        self.D = D
        self.G = self.query("total_tables")
        self.b = self.query("local_batch")
        self.out_dtype = {_lib.F32: torch.float32, _lib.BF16: torch.bfloat16,
                          _lib.F16: torch.float16}[self.get_option("out_dtype")]

    _dim_hint = 4

    def set_dim_hint(self, D: int) -> None:
        """D for a rank that registers zero tables (dim must agree across ranks)."""
        self._dim_hint = int(D)

    def forward(self, indices: torch.Tensor, offsets: torch.Tensor, stream=None,
                per_sample_weights: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Fused forward; returns a zero-copy view [b_r, G*D] of the library-owned receive buffer
        (valid until the second following forward), float32 or the "out_dtype" option's type.  per_sample_weights: optional float32 device
        tensor aligned with indices (sum pooling only)."""
        if offsets.dtype != torch.int32 or indices.dtype != torch.int32 or \
                offsets.device != self.device or indices.device != self.device or \
                not (offsets.is_contiguous() and indices.is_contiguous()):
            raise ValueError(f"indices/offsets must be contiguous int32 tensors on {self.device}")
        out, rows, cols = self._fwd_out
        n = indices.numel()
        if per_sample_weights is None:
            rc = lib.emb_a2a_forward(self._h, indices.data_ptr() if n else None,
                                     offsets.data_ptr(), n, _stream_ptr(stream, self.device),
                                     self._fwd_refs[0], self._fwd_refs[1], self._fwd_refs[2])
        else:
            _check_dev_tensor(per_sample_weights, torch.float32, "per_sample_weights", self.device)
            if per_sample_weights.numel() != n:
                raise ValueError("per_sample_weights must align with indices")
            rc = lib.emb_a2a_forward_weighted(
                self._h, indices.data_ptr() if n else None, offsets.data_ptr(),
                per_sample_weights.data_ptr() if n else None, n, _stream_ptr(stream, self.device),
                self._fwd_refs[0], self._fwd_refs[1], self._fwd_refs[2])
        if rc:
            self._err(rc, "emb_a2a_forward")
        key = (out.value or 0, rows.value, cols.value)
        v = self._views.get(key)
        if v is None:
            v = self._views[key] = _view(key[0], key[1:], self.device, self.out_dtype)
        return v

    def forward_host(self, indices: torch.Tensor, offsets: torch.Tensor, out: torch.Tensor,
                     stream=None) -> None:
        """End-to-end forward from host (pinned) int32 tensors into host float32 out [b_r, G*D];
        asynchronous on `stream` -- synchronise before reading `out`."""
        for t, dt, n in ((indices, torch.int32, "indices"), (offsets, torch.int32, "offsets"),
                         (out, self.out_dtype, "out")):
            if t.device.type != "cpu" or t.dtype != dt or not t.is_contiguous():
                raise ValueError(f"{n} must be a contiguous host {dt} tensor")
        rc = lib.emb_a2a_forward_host(self._h, indices.data_ptr() if indices.numel() else None,
                                      offsets.data_ptr(), indices.numel(),
                                      _stream_ptr(stream, self.device), out.data_ptr())
        self._err(rc, "emb_a2a_forward_host")

    # -------------------------------------------------------------- backward (f3)
    def backward_plan(self, indices: torch.Tensor, offsets: torch.Tensor, stream=None,
                      per_sample_weights: Optional[torch.Tensor] = None) -> None:
        """Sort this rank's lookups by (table, row) for the next backward (not collective).
        offsets must stay alive until that backward has run (mean pooling reads bag lengths)."""
        _check_dev_tensor(offsets, torch.int32, "offsets", self.device)
        _check_dev_tensor(indices, torch.int32, "indices", self.device)
        n = indices.numel()
        w = None
        if per_sample_weights is not None:
            _check_dev_tensor(per_sample_weights, torch.float32, "per_sample_weights", self.device)
            if per_sample_weights.numel() != n:
                raise ValueError("per_sample_weights must align with indices")
            w = per_sample_weights.data_ptr() if n else None
        self._plan_refs = (indices, offsets, per_sample_weights)
        rc = lib.emb_a2a_backward_plan(self._h, indices.data_ptr() if n else None,
                                       offsets.data_ptr(), w, n, _stream_ptr(stream, self.device))
        self._err(rc, "emb_a2a_backward_plan")

    def backward(self, grad: torch.Tensor, lr: float, stream=None) -> None:
        """Fused backward (collective): grad = dL/d(out) [b_r, G*D] float32 on this device; the
        registered tables are updated in place (sparse SGD, W -= lr * dL/dW)."""
        _check_dev_tensor(grad, torch.float32, "grad", self.device)
        if tuple(grad.shape) != (self.b, self.G * self.D):
            raise ValueError(f"grad must be [{self.b}, {self.G * self.D}]")
        rc = lib.emb_a2a_backward(self._h, grad.data_ptr() if grad.numel() else None, float(lr),
                                  _stream_ptr(stream, self.device))
        self._err(rc, "emb_a2a_backward")

    def backward_local(self, grad_mp: torch.Tensor, lr: float, stream=None) -> None:
        """Unfused second half: reduce + update from a model-parallel gradient [B, T_r, D]."""
        _check_dev_tensor(grad_mp, torch.float32, "grad_mp", self.device)
        rc = lib.emb_a2a_backward_local(self._h, grad_mp.data_ptr() if grad_mp.numel() else None,
                                        float(lr), _stream_ptr(stream, self.device))
        self._err(rc, "emb_a2a_backward_local")

    def check(self) -> None:
        """Raise if an asynchronous device failure (a wait timeout) was recorded."""
        self._err(lib.emb_a2a_check(self._h), "emb_a2a_check")

    def forward_host_batch(self, indices: Sequence[torch.Tensor], offsets: Sequence[torch.Tensor],
                           outs: Sequence[torch.Tensor], stream=None) -> None:
        """Pipelined sequence of host-buffer forwards (collective): step k reads host int32
        indices[k] / offsets[k] and writes host float32 outs[k] [b_r, G*D]; the copies of
        neighbouring steps overlap the forwards.  Synchronise `stream` before reading outs."""
        n = len(indices)
        if not (len(offsets) == n and len(outs) == n):
            raise ValueError("indices, offsets and outs must have one entry per step")
        for k in range(n):
            for t, dt, nm in ((indices[k], torch.int32, "indices"), (offsets[k], torch.int32, "offsets"),
                              (outs[k], self.out_dtype, "outs")):
                if t.device.type != "cpu" or t.dtype != dt or not t.is_contiguous():
                    raise ValueError(f"{nm}[{k}] must be a contiguous host {dt} tensor")
        P = ctypes.c_void_p * max(n, 1)
        ip = P(*[t.data_ptr() if t.numel() else None for t in indices])
        op = P(*[t.data_ptr() for t in offsets])
        outp = P(*[t.data_ptr() for t in outs])
        nn = (ctypes.c_int64 * max(n, 1))(*[t.numel() for t in indices])
        rc = lib.emb_a2a_forward_host_batch(self._h, n, ip, op, nn, outp,
                                            _stream_ptr(stream, self.device))
        self._err(rc, "emb_a2a_forward_host_batch")

    def device_barrier(self, stream=None) -> None:
        """Collective: the stream waits on the device until every rank has arrived."""
        self._err(lib.emb_a2a_device_barrier(self._h, _stream_ptr(stream, self.device)),
                  "emb_a2a_device_barrier")

    def peer_store_probe(self, bytes_per_peer: int, stream=None) -> int:
        """Bench tooling: one kernel storing into every peer's receive region at once (see
        emb_a2a.h); overwrites the peers' receive buffers.  Returns bytes written per peer."""
        used = ctypes.c_int64()
        self._err(lib.emb_a2a_peer_store_probe(self._h, int(bytes_per_peer),
                                               _stream_ptr(stream, self.device), ctypes.byref(used)),
                  "emb_a2a_peer_store_probe")
        return used.value

    def destroy(self) -> None:
        if self._h:
            rc = lib.emb_a2a_destroy(self._h)
            self._h = ctypes.c_void_p()
            self._tables = []
            if rc:
                raise EmbA2AError(rc, "emb_a2a_destroy")

    # -------------------------------------------------------------- local API
    def pool_local(self, indices: torch.Tensor, offsets: torch.Tensor, send: torch.Tensor,
                   stream=None, per_sample_weights: Optional[torch.Tensor] = None) -> None:
        """Unfused baseline first half: send [B, T_r, D] of the output type (dest-major blocks by
        p_s)."""
        _check_dev_tensor(send, self.out_dtype, "send", self.device)
        _check_dev_tensor(offsets, torch.int32, "offsets", self.device)
        _check_dev_tensor(indices, torch.int32, "indices", self.device)
        n = indices.numel()
        w = None
        if per_sample_weights is not None:
            _check_dev_tensor(per_sample_weights, torch.float32, "per_sample_weights", self.device)
            w = per_sample_weights.data_ptr() if n else None
        rc = lib.emb_a2a_pool_local_weighted(self._h, indices.data_ptr() if n else None,
                                             offsets.data_ptr(), w, n,
                                             _stream_ptr(stream, self.device), send.data_ptr())
        self._err(rc, "emb_a2a_pool_local")

    def set_option(self, key: str, value: int) -> None:
        self._err(lib.emb_a2a_set_option(self._h, key.encode(), int(value)), f"set_option({key})")

    def get_option(self, key: str) -> int:
        v = ctypes.c_int64()
        self._err(lib.emb_a2a_get_option(self._h, key.encode(), ctypes.byref(v)), f"get_option({key})")
        return v.value

    def query(self, key: str) -> int:
        v = ctypes.c_int64()
        self._err(lib.emb_a2a_query(self._h, key.encode(), ctypes.byref(v)), f"query({key})")
        return v.value

    def slice_plan(self) -> np.ndarray:
        n = self.query("num_slices")
        out = np.zeros((max(n, 1), 4), dtype=np.int32)
        nn = ctypes.c_int64()
        self._err(lib.emb_a2a_slice_plan(self._h, out.ctypes.data, n, ctypes.byref(nn)),
                  "emb_a2a_slice_plan")
        return out[:n]

    def read_trace(self) -> np.ndarray:
        """Per-CTA timeline since the last read: structured array (cta, event, payload, t_ns)."""
        cap = self.get_option("trace")
        buf = np.zeros((max(cap, 1), 2), dtype=np.uint64)
        n = ctypes.c_int64()
        self._err(lib.emb_a2a_read_trace(self._h, buf.ctypes.data, cap, ctypes.byref(n)),
                  "emb_a2a_read_trace")
        buf = buf[: n.value]
        out = np.zeros(n.value, dtype=[("cta", "i4"), ("event", "i4"), ("payload", "i8"),
                                       ("t_ns", "i8")])
        out["cta"] = (buf[:, 0] >> np.uint64(40)).astype(np.int64)
        out["event"] = ((buf[:, 0] >> np.uint64(32)) & np.uint64(0xFF)).astype(np.int64)
        out["payload"] = (buf[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.int64)
        out["t_ns"] = buf[:, 1].astype(np.int64)
        return out

    def read_flags(self) -> np.ndarray:
        out = np.zeros(self.W, dtype=np.uint64)
        self._err(lib.emb_a2a_read_flags(self._h, out.ctypes.data, self.W), "emb_a2a_read_flags")
        return out

    def __del__(self):   # best effort; destroy() is collective and should be called explicitly
        pass


def run_ranks(fn: Callable[[int], object], world_size: int) -> list:
    """Run fn(rank) on world_size host threads (for collective calls on virtual ranks)."""
    results: list = [None] * world_size
    errors: list = [None] * world_size

    def body(r):
        try:
            results[r] = fn(r)
        except BaseException as e:      # re-raised below
            errors[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(world_size)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errors:
        if e is not None:
            raise e
    return results
