"""W virtual ranks of the fused op on ONE device (single-GPU loopback, SURVEY.md Sec 4 tier T1).

Each virtual rank is a full EmbA2A handle with its own symmetric region; "peer" pointers are
same-process raw pointers, so the kernels, counters and waits are exactly the multi-GPU ones
with NVLink replaced by local HBM.  Forwards go on W separate streams so the W fused kernels
can be co-resident (a rank's receive wait needs its peers' kernels to make progress).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from .emb_a2a import EmbA2A, LocalGroup, run_ranks


class LoopbackGroup:
    def __init__(self, world_size: int, device="cuda:0", options: Optional[dict] = None):
        self.W = world_size
        self.device = torch.device(device)
        self.group = LocalGroup(world_size)
        self.handles: List[EmbA2A] = [
            EmbA2A(r, world_size, self.device, self.group.allgather_for(r), options)
            for r in range(world_size)]
        self.streams = [torch.cuda.Stream(self.device) for _ in range(world_size)]

    def set_option(self, key: str, value: int) -> None:
        for h in self.handles:
            h.set_option(key, value)

    def register_tables(self, tables: Sequence[Sequence[torch.Tensor]], global_batch: int,
                        partition: Optional[Sequence[int]] = None, dim: Optional[int] = None,
                        pooling: str = "sum", dtype: Optional[torch.dtype] = None):
        if dim is not None:
            for h in self.handles:
                h.set_dim_hint(dim)
        run_ranks(lambda r: self.handles[r].register_tables(tables[r], global_batch, partition,
                                                            pooling, dtype), self.W)

    def forward(self, indices: Sequence[torch.Tensor], offsets: Sequence[torch.Tensor],
                sync: bool = True, weights: Optional[Sequence[torch.Tensor]] = None,
                aligned: bool = False) -> List[torch.Tensor]:
        """aligned: put a cross-rank device barrier in front of the W forwards so the virtual
        ranks start together (the host issues them one after another)."""
        cur = torch.cuda.current_stream(self.device)
        outs = []
        if aligned:   # hold the GPU long enough for the host to enqueue all W forwards
            torch.cuda._sleep(4_000_000)
        for r, h in enumerate(self.handles):
            self.streams[r].wait_stream(cur)
        if aligned:
            for r, h in enumerate(self.handles):
                h.device_barrier(self.streams[r])
        for r, h in enumerate(self.handles):
            outs.append(h.forward(indices[r], offsets[r], stream=self.streams[r],
                                  per_sample_weights=None if weights is None else weights[r]))
        for s in self.streams:
            cur.wait_stream(s)
        if sync:
            torch.cuda.synchronize(self.device)
        return outs

    def backward(self, indices: Sequence[torch.Tensor], offsets: Sequence[torch.Tensor],
                 grads: Sequence[torch.Tensor], lr: float, sync: bool = True,
                 weights: Optional[Sequence[torch.Tensor]] = None, plan: bool = True) -> None:
        """Plan (sort) + fused backward on every virtual rank, W streams.  The backward's
        persistent grid is shared W+1 ways so all W kernels are resident together with room to
        spare (each waits for the others' gradient rows)."""
        cur = torch.cuda.current_stream(self.device)
        share = self.W + 1 if self.W > 1 else 1   # slack: the grids must co-reside exactly
        for r, h in enumerate(self.handles):
            if h.get_option("bwd_share") != share:
                h.set_option("bwd_share", share)
            self.streams[r].wait_stream(cur)
        if plan:
            for r, h in enumerate(self.handles):
                h.backward_plan(indices[r], offsets[r], stream=self.streams[r],
                                per_sample_weights=None if weights is None else weights[r])
            # every plan before any backward: on ONE device the W persistent backward grids fill
            # the GPU while they wait for each other's gradient rows, so a plan still queued
            # behind them could never get an SM (on W GPUs each plan has its own device)
            done = [torch.cuda.Event() for _ in range(self.W)]
            for r in range(self.W):
                done[r].record(self.streams[r])
            for r in range(self.W):
                for e in done:
                    self.streams[r].wait_event(e)
        for r, h in enumerate(self.handles):
            h.backward(grads[r], lr, stream=self.streams[r])
        for s in self.streams:
            cur.wait_stream(s)
        if sync:
            torch.cuda.synchronize(self.device)
            for h in self.handles:
                h.check()

    def destroy(self):
        run_ranks(lambda r: self.handles[r].destroy(), self.W)
